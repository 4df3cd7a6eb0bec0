#!/bin/bash
# (historical: measured and reverted; the variant and its knob are no longer in the tree -- DESIGN §5.1)
# lane-major 4-step slot-word groups (one 8-byte load per batch)
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x --timeout 800 > gpurun_out/wg_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/wg_tests.log
for c in c5 c3 c5; do
  SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/wg_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/wg_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('$c value %.2f e2e %.2f A %.3f At %.3f frac %.3f sm %s' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['roofline']['frac'], d['clocks']['sm_mhz']))"
done
