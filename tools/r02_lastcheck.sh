#!/bin/bash
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 2300 > gpurun_out/lc_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/lc_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lc_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/lc_smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/lc_ref.log 2> gpurun_out/lc_ref.err; echo ref_rc=$?; tail -c 600 gpurun_out/lc_ref.log
