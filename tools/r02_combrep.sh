#!/bin/bash
# in-graph cost of the split combines: iteration time with each combine launched 1x / 2x / 3x
for rep in 1 2 3 1; do
for c in c3 c5; do
  SCS_COMBINE_REPEAT=$rep SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/cr${rep}_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/cr${rep}_$c.log').read().strip().splitlines()[-1])
print('rep=$rep $c value %.2f ms/it %.4f sm %s' % (d['value'], 1e3/d['value'], d['clocks']['sm_mhz']))"
done
done
