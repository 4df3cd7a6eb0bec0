#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/r02_gpu4_tests.log 2>&1; echo tests_rc=$?
tail -6 gpurun_out/r02_gpu4_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench4.log 2> gpurun_out/r02_bench4.err; echo bench_rc=$?
tail -3 gpurun_out/r02_bench4.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench4.log').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],'r32',d['value_r32']['value'],'frac',d['roofline']['frac']); print(json.dumps(d['roofline']['kernels']))"
SCS_BENCH_CONFIG=c3 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-optin --no-cpu > gpurun_out/r02_bench4_c3.log 2>&1; echo c3_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench4_c3.log').read().strip().splitlines()[-1])
print('c3 value',d['value'],'e2e',d['e2e']['value'],'frac',d['roofline']['frac']); print(json.dumps(d['roofline']['kernels'])); print(d.get('time_to_eps',{}).get('time_to_eps_s'))"
export SCS_LOOP_GRAPH=0
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_c5_launches4.csv python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_ncu_list4.log 2>&1; echo list_rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_stream -c 3 -o gpurun_out/r02_c5_stream_v3 -f python tools/ncu_iteration.py c5 --kernels > gpurun_out/r02_ncu_full4.log 2>&1; echo full_rc=$?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_c3_launches4.csv python tools/ncu_iteration.py c3 --kernels > gpurun_out/r02_ncu_list4c3.log 2>&1; echo list3_rc=$?
