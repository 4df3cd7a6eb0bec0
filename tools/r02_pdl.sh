#!/bin/bash
for v in 0 1 0 1; do SCS_PDL=$v timeout 300 python tools/ncu_c1.py 2>&1 | tail -1 | sed "s/^/pdl=$v /"; done
SCS_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -q -x --timeout 800 > gpurun_out/pdl_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/pdl_tests.log
for v in 0 1; do
  SCS_PDL=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/pdl_c5_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/pdl_c5_$v.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('pdl=$v c5 value %.2f e2e %.2f' % (d['value'], d['e2e']['value']))"
done
