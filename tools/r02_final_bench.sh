#!/bin/bash
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/rf_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/rf_bench.log 2> gpurun_out/rf_bench.err; echo bench_rc=$?
tail -2 gpurun_out/rf_bench.err
SCS_BENCH_CONFIG=c3 timeout 900 python bench.py --steps 20 --warmup 5 --no-configs > gpurun_out/rf_bench_c3.log 2> gpurun_out/rf_bench_c3.err; echo c3_rc=$?
