"""Time the device PSD projection (scs_project_cone, one call = handle setup +
H2D + projection + D2H) at large sides, cooperative-grid Jacobi vs the r01
one-CTA path (SCS_PSD_GRID=0).  Usage: python tools/psd_bench.py [sides...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1312_3039_b200 import native  # noqa: E402

sides = [int(a) for a in sys.argv[1:]] or [256, 500, 1000, 2000]
old_max = int(os.environ.get("PSD_BENCH_OLD_MAX", "0"))
for k in sides:
    rng = np.random.default_rng(k)
    x = rng.standard_normal(k * (k + 1) // 2)
    row = {"side": k}
    for mode in ("1", "0"):
        if mode == "0" and k > old_max:
            continue
        os.environ["SCS_PSD_GRID"] = mode
        native.project_cone(x[:3], {"s": [2]})  # context warm-up
        ts = []
        for _ in range(3 if mode == "1" else 1):
            t0 = time.perf_counter()
            native.project_cone(x, {"s": [k]})
            ts.append(time.perf_counter() - t0)
        row["grid_s" if mode == "1" else "cta_s"] = round(min(ts), 4)
    print(row, flush=True)
