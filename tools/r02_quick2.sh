#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_production.py -q -x --timeout 800 > gpurun_out/q2_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/q2_tests.log
for cap in default 32768 20480; do
  if [ $cap = default ]; then unset SCS_STREAM_CAP; else export SCS_STREAM_CAP=$cap; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/q2_$cap.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/q2_$cap.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('cap=$cap value %.2f e2e %.2f A %.3f At %.3f' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms']))"
done
