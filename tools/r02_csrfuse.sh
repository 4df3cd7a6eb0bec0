#!/bin/bash
# CSR path: first A^T pass with its epilogue in k_spmv (no Sv + k_rows), final A pass as EpiAFinal
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_resrec.py tests/test_gpu_c4.py tests/test_gpu_sharded.py tests/test_gpu_optin.py tests/test_gpu_check.py -q -x --timeout 2300 > gpurun_out/cf_tests.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/cf_tests.log
SCS_LOOP_GRAPH=0 timeout 300 python tools/ncu_c4.py > gpurun_out/cf_c4.log 2>&1; tail -1 gpurun_out/cf_c4.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-tte --no-optin --no-cpu > gpurun_out/cf_bench.log 2>&1; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/cf_bench.log').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'])
for k,v in d['baseline_configs'].items(): print(k, v.get('status'), v.get('iterations'), v.get('us_per_iter'))"
