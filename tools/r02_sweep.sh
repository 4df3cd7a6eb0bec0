#!/bin/bash
# streamed-format sweep at C5: slab width x piece cap (stages = smem left / cap, <= 8)
for wc in "4096 32768" "4096 24576" "4096 16384" "2048 32768" "2048 16384" "2048 24576"; do
  set -- $wc
  SCS_STREAM_W=$1 SCS_STREAM_CAP=$2 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/sw_$1_$2.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/sw_$1_$2.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('W=$1 cap=$2 value %.2f A %.3f At %.3f' % (d['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms']))"
done
