#!/bin/bash
timeout 400 python -m pytest tests/test_gpu_bands.py -q -x --timeout 200 -o timeout_method=thread > gpurun_out/pytest_bands.log 2>&1; echo bands_rc=$?; tail -3 gpurun_out/pytest_bands.log
for B in 1 5 3 8; do
  SCS_DEBUG=1 SCS_BANDS=$B timeout 600 python bench.py --config c5 --steps 20 --no-cpu --no-tte > gpurun_out/bench_b$B.log 2> gpurun_out/bench_b$B.err; echo b${B}_rc=$?
  grep -E "bands:" gpurun_out/bench_b$B.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_b$B.log').read().strip().splitlines()[-1]); r=d['roofline']
print('B=$B', round(d['value'],2), round(d['ms_per_step'],3), {k[:8]:(round(v['ms'],3),round(v['gbs'])) for k,v in r['kernels'].items()})"
done
