#!/bin/bash
# roofline kernel timing: interleaved A / A^T rounds, median
for i in 1 2; do for c in c5 c3; do
  SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/rs_${c}_$i.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/rs_${c}_$i.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('$c value %.2f frac %.3f A %s At %s sm %s' % (d['value'], d['roofline']['frac'], k['spmv_A(q=A p)']['ms_samples'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms_samples'], d['clocks']['sm_mhz']))"
done; done
