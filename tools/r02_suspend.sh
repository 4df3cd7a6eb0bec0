#!/bin/bash
# mbarrier try_wait suspend-time hint: 500 / 2000 (kept) / 8000 ns
cp paper_1312_3039_b200/libscs_b200.so /tmp/lib_keep.so
for v in s2000 s500 s8000 s2000 s500 s8000; do
  cp tools/_ab/lib_$v.so paper_1312_3039_b200/libscs_b200.so
  SCS_BENCH_CONFIG=c5 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/su_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/su_$v.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('$v c5 value %.2f A %.3f At %.3f sm %s' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
done
cp /tmp/lib_keep.so paper_1312_3039_b200/libscs_b200.so
