#!/bin/bash
# r02 third GPU pass: format v2 -- stream/parity/production/multiproc tests, C5 setup debug, bench, ncu
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_production.py tests/test_gpu_multiproc.py tests/test_gpu_parity.py tests/test_gpu_resrec.py tests/test_gpu_sharded.py -q -rf --timeout 1200 -x > gpurun_out/r02_gpu3_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r02_gpu3_tests.log
SCS_DEBUG=1 timeout 300 python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_c5_debug.log 2>&1; echo dbg_rc=$?
grep -E "stream (pin|layout|sched)|graphs" gpurun_out/r02_c5_debug.log | head -20
timeout 900 python bench.py --steps 20 --warmup 5 --no-configs > gpurun_out/r02_bench3.log 2> gpurun_out/r02_bench3.err; echo bench_rc=$?
tail -c 1200 gpurun_out/r02_bench3.log; tail -3 gpurun_out/r02_bench3.err
export SCS_LOOP_GRAPH=0
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_stream -c 3 -o gpurun_out/r02_c5_stream_v2 -f python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_ncu_full3.log 2>&1; echo full_rc=$?
tail -2 gpurun_out/r02_ncu_full3.log
