#!/bin/bash
# one iteration of config ${CFG:-c5}: launch list + full capture of the streamed SpMV kernels
CFG=${CFG:-c5}
timeout 300 python tools/ncu_iteration.py $CFG --kernels > gpurun_out/ncu_plain_$CFG.log 2>&1; rc=$?; echo plain_rc=$rc; tail -2 gpurun_out/ncu_plain_$CFG.log
[ $rc -eq 0 ] || exit 1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/${CFG}_iter_stm.csv python tools/ncu_iteration.py $CFG > gpurun_out/ncu_list_$CFG.log 2>&1; echo list_rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_stream -o gpurun_out/${CFG}_stm_full -f python tools/ncu_iteration.py $CFG > gpurun_out/ncu_full_$CFG.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full_$CFG.log
