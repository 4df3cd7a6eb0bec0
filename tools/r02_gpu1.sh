#!/bin/bash
# r02 first GPU pass: full GPU suite (new production-scale + golden parity tests), smoke, default bench
nvidia-smi --query-gpu=name,memory.total --format=csv,noheader
free -g | head -2; nproc
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/r02_gpu1_tests.log 2>&1; echo tests_rc=$?
tail -25 gpurun_out/r02_gpu1_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r02_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench1.log 2> gpurun_out/r02_bench1.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r02_bench1.log; tail -5 gpurun_out/r02_bench1.err
