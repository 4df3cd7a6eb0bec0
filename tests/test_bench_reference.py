"""The CPU reference arm of bench.py (CPU only): the contract's JSON line,
and no library of this repository mapped into the process -- the reference
arm must time the reference algorithm alone (the port of conesplit's path on
numpy, data from the numpy twin of the native generator)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_and_no_repo_library():
    env = dict(os.environ, SCS_BENCH_REF_CONFIG="tiny", OPENBLAS_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "3", "--warmup", "3", "--no-configs"], env=env,
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 3 and line["warmup"] == 3
    assert line["value"] > 0 and line["unit"] == "iters/s" and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"] == "lasso_socp_tiny"
    assert line["extrapolated"]["config"] == "lasso_socp_c5"
    assert line["repo_libs_loaded"] == []
