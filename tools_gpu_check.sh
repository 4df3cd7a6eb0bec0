#!/bin/bash
# quick GPU validation: smoke, gpu tests, c3/c5 bench lines (no CPU baseline)
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -o timeout_method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "^(FAILED|ERROR)|passed|failed|Error |assert" gpurun_out/pytest_gpu.log | head -30
for cfg in ${CFGS:-c3 c5}; do
  timeout 600 python bench.py --config $cfg --steps 20 --no-cpu --no-tte > gpurun_out/bench_$cfg.log 2>&1; echo ${cfg}_rc=$?
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_c*.log")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, round(d["value"], 2), "it/s", round(d["ms_per_step"], 3), "ms", "kfrac", round(r["frac"], 3),
              "iterfrac", round(r["iteration"]["frac"], 3),
              {k[:8]: (round(v["ms"], 3), round(v["gbs"])) for k, v in r["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-800:])
PY
