#!/bin/bash
# k_psd_small with the side as a template constant (switch dispatch)
export SCS_LOOP_GRAPH_SAVE=$SCS_LOOP_GRAPH
timeout 1200 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py tests/test_gpu_psd_large.py -q -x --timeout 1100 > gpurun_out/kc_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/kc_tests.log
SCS_LOOP_GRAPH=0 timeout 300 python tools/ncu_c4.py > gpurun_out/kc_c4_plain.log 2>&1; echo c4_rc=$?; tail -1 gpurun_out/kc_c4_plain.log
SCS_LOOP_GRAPH=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kc_c4_launches.csv python tools/ncu_c4.py > gpurun_out/kc_c4_ncu.log 2>&1; echo c4ncu_rc=$?
