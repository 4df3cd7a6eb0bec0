#!/bin/bash
# final one-iteration launch lists, configs 5 and 3 (steady state, non-refresh iteration)
export SCS_LOOP_GRAPH=0
for c in c5 c3; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/fl_$c.csv python tools/ncu_iteration.py $c --kernels > gpurun_out/fl_$c.log 2>&1; echo list_rc=$?
done
