#!/bin/bash
# one C5 iteration: plain run, launch list with DRAM bytes, full capture of the SpMV kernels
timeout 300 python tools/ncu_iteration.py c5 --kernels > gpurun_out/ncu_plain.log 2>&1; rc=$?; echo plain_rc=$rc; tail -2 gpurun_out/ncu_plain.log
[ $rc -eq 0 ] || exit 1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/c5_iter.csv python tools/ncu_iteration.py c5 --kernels > gpurun_out/ncu_list.log 2>&1; echo list_rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_spmv -o gpurun_out/c5_full -f python tools/ncu_iteration.py c5 > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full.log
