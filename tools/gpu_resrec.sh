#!/bin/bash
# residual recurrence: new tests, full GPU suite, bench lines (c5, c3) with R=32 and R=0
timeout 600 python -m pytest tests/test_gpu_resrec.py -q -x --timeout 300 -o timeout_method=thread > gpurun_out/pytest_resrec.log 2>&1; echo resrec_rc=$?
tail -3 gpurun_out/pytest_resrec.log; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/pytest_resrec.log | head -20
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -o timeout_method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 600 python bench.py --no-cpu --no-tte --no-optin > gpurun_out/bench_c5_rr.log 2> gpurun_out/bench_c5_rr.err; echo c5_rc=$?
SCS_RES_RECUR=0 timeout 600 python bench.py --no-cpu --no-tte --no-optin > gpurun_out/bench_c5_rr0.log 2> gpurun_out/bench_c5_rr0.err; echo c50_rc=$?
timeout 600 python bench.py --config c3 --no-cpu --no-tte --no-optin > gpurun_out/bench_c3_rr.log 2> gpurun_out/bench_c3_rr.err; echo c3_rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5_rr.log", "gpurun_out/bench_c5_rr0.log", "gpurun_out/bench_c3_rr.log"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"], 2), "it/s", round(d["ms_per_step"], 3), "ms e2e", round(d["e2e"]["value"], 2), "launches/step", d.get("launches_per_step"), d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
