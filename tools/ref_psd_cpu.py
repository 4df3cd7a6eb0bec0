"""Time the REFERENCE's PSD projection (conesplit cones._project_psd: numba
cyclic Jacobi, _kernels.py:119-191) on this container's CPU, for the
large-PSD comparison in DESIGN.md.  Build container only (imports
/root/reference).  Usage: python tools/ref_psd_cpu.py [sides...]"""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from conesplit import cones  # noqa: E402

cones._project_psd(np.ones(3), 2)  # numba compile
for k in [int(a) for a in sys.argv[1:]] or [200, 500, 1000]:
    x = np.random.default_rng(k).standard_normal(k * (k + 1) // 2)
    t = time.perf_counter()
    cones._project_psd(x, k)
    print({"side": k, "reference_cpu_s": round(time.perf_counter() - t, 3)}, flush=True)
