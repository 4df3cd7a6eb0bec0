#!/bin/bash
# r02 second GPU pass: full GPU suite, smoke, default bench, C5 launch list + full capture of the streamed SpMV
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/r02_gpu2_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r02_gpu2_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke2.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r02_smoke2.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench2.log 2> gpurun_out/r02_bench2.err; echo bench_rc=$?
tail -c 1500 gpurun_out/r02_bench2.log; tail -5 gpurun_out/r02_bench2.err
export SCS_LOOP_GRAPH=0
timeout 300 python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_ncu_plain.log 2>&1; rc=$?; echo plain_rc=$rc
[ $rc -eq 0 ] || exit 1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_c5_launches.csv python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_ncu_list.log 2>&1; echo list_rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_stream -o gpurun_out/r02_c5_stream_full -f python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_ncu_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/r02_ncu_full.log
