#!/bin/bash
# stream gate at 4e6 nonzeros: heuristic tests, every stream / parity / production test, the s1e7 bench config
timeout 2400 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_resrec.py tests/test_gpu_optin.py tests/test_gpu_sharded.py tests/test_gpu_c4.py -q -x --timeout 2300 > gpurun_out/ga_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/ga_tests.log
for c in s1e7 c3; do
  SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/ga_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ga_$c.log').read().strip().splitlines()[-1])
print('$c value %.2f e2e %.2f' % (d['value'], d['e2e']['value']))"
  SCS_STREAM=0 SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/ga0_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ga0_$c.log').read().strip().splitlines()[-1])
print('$c CSR value %.2f e2e %.2f' % (d['value'], d['e2e']['value']))"
done
