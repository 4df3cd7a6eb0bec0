#!/bin/bash
# A/B: the library at 62c5bab vs now, configs 3 and 5 on the same box
cp paper_1312_3039_b200/libscs_b200.so /tmp/lib_keep.so
for v in old new old new; do
  cp tools/_ab/lib_$v.so paper_1312_3039_b200/libscs_b200.so
  for c in c3 c5; do
    SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/abc_${v}_$c.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/abc_${v}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('$v $c value %.2f A %.3f At %.3f sm %s' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
  done
done
cp /tmp/lib_keep.so paper_1312_3039_b200/libscs_b200.so
