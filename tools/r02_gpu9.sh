#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/r02_gpu9_tests.log 2>&1; echo tests_rc=$?
tail -4 gpurun_out/r02_gpu9_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r9_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r9_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r9_bench.log 2> gpurun_out/r9_bench.err; echo bench_rc=$?
SCS_BENCH_CONFIG=c3 timeout 900 python bench.py --steps 20 --warmup 5 --no-configs > gpurun_out/r9_bench_c3.log 2> gpurun_out/r9_bench_c3.err; echo c3_rc=$?
export SCS_LOOP_GRAPH=0
for c in c5 c3; do
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r9_launches_$c.csv python tools/ncu_iteration.py $c --kernels > gpurun_out/r9_list_$c.log 2>&1; echo list_rc=$?
done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_stream -c 3 -o gpurun_out/r9_c5_stream -f python tools/ncu_iteration.py c5 --kernels > gpurun_out/r9_ncu_full.log 2>&1; echo full_rc=$?
