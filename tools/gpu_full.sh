#!/bin/bash
# full GPU validation + default bench line + c3 line
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -o timeout_method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench_rc=$?
timeout 600 python bench.py --config c3 --steps 50 --no-cpu --no-tte > gpurun_out/bench_c3.log 2> gpurun_out/bench_c3.err; echo c3_rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_default.log", "gpurun_out/bench_c3.log"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, round(d["value"], 2), "it/s", round(d["ms_per_step"], 3), "ms kfrac", round(r["frac"], 3),
              "iterfrac", round(r["iteration"]["frac"], 3), "e2e", round(d["e2e"]["value"], 2),
              "optin", d.get("opt_in"), "tte", {k: d.get("time_to_eps", {}).get(k) for k in ("iterations", "time_to_eps_s")},
              "tte_optin", d.get("time_to_eps", {}).get("opt_in"), "clocks", d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
