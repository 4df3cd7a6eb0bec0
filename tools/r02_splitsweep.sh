#!/bin/bash
# A^T split count at config 5 / 3 (the model's choice is printed by SCS_DEBUG)
SCS_DEBUG=1 SCS_BENCH_CONFIG=c5 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/ss_def_c5.log 2> gpurun_out/ss_def_c5.err
grep "stream sched" gpurun_out/ss_def_c5.err | head -4
for sp in def 4 8 24 def; do
  for c in c5; do
    if [ $sp = def ]; then unset SCS_STREAM_SPLITS_AT; else export SCS_STREAM_SPLITS_AT=$sp; fi
    SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/ss_${sp}_$c.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ss_${sp}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('at_splits=$sp $c value %.2f A %.3f At %.3f sm %s' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
  done
done
