#!/bin/bash
# quick perf probe: C5 bench line (no tte/configs/cpu) + one full ncu capture of the A^T CG pass
timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/q_bench.log 2> gpurun_out/q_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/q_bench.log').read().strip().splitlines()[-1])
print('value',d['value'],'e2e',d['e2e']['value'],'r32',d['value_r32']['value']); print(json.dumps(d['roofline']['kernels']))"
export SCS_LOOP_GRAPH=0
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:EpiAtGp -c 1 -o gpurun_out/q_ncu -f python tools/ncu_iteration.py ${1:-c5} > gpurun_out/q_ncu.log 2>&1; echo ncu_rc=$?
