#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_c4.py tests/test_gpu_parity.py tests/test_gpu_psd_large.py tests/test_gpu_check.py tests/test_gpu_optin.py -q -x --timeout 1400 > gpurun_out/pf_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/pf_tests.log
SCS_LOOP_GRAPH=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pf_c4_launches.csv python tools/ncu_c4.py > gpurun_out/pf_c4_ncu.log 2>&1; echo c4ncu_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --no-tte --no-optin --no-cpu > gpurun_out/pf_bench.log 2>&1; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/pf_bench.log').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value']); print(json.dumps(d.get('baseline_configs'))[:3000])"
