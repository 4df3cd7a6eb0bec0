#!/bin/bash
export SCS_LOOP_GRAPH=0
for c in c3 c5; do
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/rl_$c.csv python tools/ncu_iteration.py $c --kernels > gpurun_out/rl_$c.log 2>&1; echo list_rc=$?
done
