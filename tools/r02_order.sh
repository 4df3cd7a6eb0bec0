#!/bin/bash
# each CTA's split parts in slab-range order (SCS_STREAM_ORDER=1) vs LPT assignment order (0)
for o in 1 0 1 0; do
  for c in c5 c3; do
    SCS_STREAM_ORDER=$o SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/or${o}_$c.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/or${o}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('order=$o $c value %.2f A %.3f At %.3f sm %s' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
  done
done
