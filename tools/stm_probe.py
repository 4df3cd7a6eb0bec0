"""Streamed-tile self-check on small random matrices under env variants
(SCS_STREAM_CHECK=1 prints streamed vs CSR product differences)."""
import os, subprocess, sys
VARS = [{}, {"SCS_STREAM_SPLITS": "1"}, {"SCS_STREAM_CAP": "200000"}, {"SCS_STREAM_W": "64"},
        {"SCS_STREAM_W": "512", "SCS_STREAM_CAP": "6208"}]
CODE = r'''
import numpy as np, sys
sys.path.insert(0, ".")
import paper_1312_3039_b200 as P
m, n, dens = %s
rng = np.random.default_rng(m + n)
nnz = max(1, int(dens * m * n))
lin = np.unique(rng.integers(0, m * n, nnz))
cols, rows = np.divmod(lin, m)
vals = rng.standard_normal(lin.size)
colptr = np.zeros(n + 1, np.int64); np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n), P.ConeSpec(nonneg_dim=m))
try:
    P.Workspace(data, P.Settings(normalize=False))
    print("create ok")
except Exception as e:
    print("create failed:", e)
'''
for shape in ["(3000, 1000, 0.01)", "(3000, 1000, 0.001)", "(9000, 200, 0.05)"]:
    for v in VARS:
        env = dict(os.environ, SCS_STREAM="1", SCS_STREAM_CHECK="1", SCS_DEBUG="1", **v)
        r = subprocess.run([sys.executable, "-c", CODE % shape], env=env, capture_output=True, text=True, timeout=120)
        print("=== shape", shape, v)
        for line in (r.stdout + r.stderr).splitlines():
            if "stream" in line or "create" in line or "Error" in line:
                print("   ", line)
