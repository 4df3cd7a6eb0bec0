#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q -x --timeout 300 -o timeout_method=thread > gpurun_out/pytest_stream.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_stream.log; grep -E "^(FAILED|ERROR)|Error|assert " gpurun_out/pytest_stream.log | head -10
SCS_DEBUG=1 timeout 900 python bench.py --steps 20 --no-cpu --no-tte --no-optin > gpurun_out/bench_c5_stm.log 2> gpurun_out/bench_c5_stm.err; echo c5_rc=$?
grep -E "stream" gpurun_out/bench_c5_stm.err | head; tail -3 gpurun_out/bench_c5_stm.err
SCS_STREAM=1 timeout 600 python bench.py --config c3 --steps 50 --no-cpu --no-tte --no-optin > gpurun_out/bench_c3_stm.log 2> gpurun_out/bench_c3_stm.err; echo c3_rc=$?
python3 - <<'PY'
import json
for f in ['gpurun_out/bench_c3_stm.log','gpurun_out/bench_c5_stm.log']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r=d['roofline']
        print(f, round(d['value'],2), round(d['ms_per_step'],3), {k:(round(v['ms'],3), round(v['gbs'])) for k,v in r['kernels'].items()})
    except Exception as e: print(f, "ERR", e)
PY
