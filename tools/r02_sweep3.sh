#!/bin/bash
for cfg in "0 3" "0 4" "1 3" "1 4" "0 5"; do
  set -- $cfg
  SCS_STREAM_PAIR=$1 SCS_STREAM_STAGES=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/sw3_$1_$2.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/sw3_$1_$2.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('pair=$1 stages=$2 value %.2f A %.3f At %.3f' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms']))"
done
