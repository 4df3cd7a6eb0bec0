#!/bin/bash
# long split rows summed inside k_rows (no k_seg_long launch)
timeout 1500 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_check.py -q -x --timeout 1400 > gpurun_out/sl_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/sl_tests.log
SCS_LOOP_GRAPH=0 timeout 300 python tools/ncu_c4.py > gpurun_out/sl_c4.log 2>&1; tail -1 gpurun_out/sl_c4.log
SCS_LOOP_GRAPH=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sl_c4_launches.csv python tools/ncu_c4.py > gpurun_out/sl_c4_ncu.log 2>&1; echo c4ncu_rc=$?
