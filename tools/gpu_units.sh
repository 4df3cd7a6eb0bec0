#!/bin/bash
for U in 16; do
for C in c3 c5; do
SCS_STREAM_UNITS=$U timeout 900 python bench.py --config $C --steps 30 --no-cpu --no-tte --no-optin > gpurun_out/b_${C}_$U.log 2>/dev/null
python3 - <<PY
import json
d=json.loads(open('gpurun_out/b_${C}_$U.log').read().strip().splitlines()[-1])
print('$C units $U', round(d['value'],2), round(d['ms_per_step'],3))
PY
done; done
