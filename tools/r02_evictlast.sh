#!/bin/bash
# (historical: measured and reverted; the variant is no longer in the tree -- DESIGN §5.1)
# gather-vector slab copies with an L2 evict_last policy (el1) vs no hint (el0)
cp paper_1312_3039_b200/libscs_b200.so /tmp/lib_keep.so
for v in el1 el0 el1 el0; do
  cp tools/_ab/lib_$v.so paper_1312_3039_b200/libscs_b200.so
  for c in c5 c3; do
    SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/el_${v}_$c.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/el_${v}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('$v $c value %.2f A %.3f At %.3f sm %s' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
  done
done
cp /tmp/lib_keep.so paper_1312_3039_b200/libscs_b200.so
