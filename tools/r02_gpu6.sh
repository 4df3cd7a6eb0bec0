#!/bin/bash
for v in "1 c5" "0 c5" "1 c3" "0 c3"; do
  set -- $v
  SCS_STREAM_COOP=$1 SCS_BENCH_CONFIG=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/q6_$1_$2.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/q6_$1_$2.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('coop=$1 $2 value %.2f A %.3f At %.3f' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms']))"
done
