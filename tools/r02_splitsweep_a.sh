#!/bin/bash
# A split count at config 3 (model: 4), iteration rate and the A pass
for sp in def 2 3 6 def 2; do
  if [ $sp = def ]; then unset SCS_STREAM_SPLITS_A; else export SCS_STREAM_SPLITS_A=$sp; fi
  SCS_BENCH_CONFIG=c3 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/ssa_${sp}.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ssa_${sp}.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('a_splits=$sp c3 value %.2f A %.4f At %.4f' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms']))"
done
