#!/bin/bash
# default bench line + C5 one-iteration launch list (no full capture)
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout 300 python tools/ncu_iteration.py c5 --kernels > gpurun_out/ncu_plain_c5.log 2>&1; rc=$?; echo plain_rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/c5_iter_rr.csv python tools/ncu_iteration.py c5 > gpurun_out/ncu_list_c5.log 2>&1; echo list_rc=$?
