"""Streamed tiles vs the CSR kernel on sparse shapes at >= 2e7 nonzeros:
device-timed us/iteration of a few ADMM iterations (scs_bench_iters) with
SCS_STREAM=1 and SCS_STREAM=0 (read at Workspace creation)."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import native


def problem(m, n, nz, seed):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, m, nz)
    cols = rng.integers(0, n, nz)
    key = np.unique(cols.astype(np.int64) * m + rows)
    cols, rows = np.divmod(key, m)
    vals = rng.standard_normal(key.size)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    # LP rows: A x + s = b, s >= 0 (a feasible, bounded-ish instance is not needed for timing)
    return P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))


def timed(data, stream):
    os.environ["SCS_STREAM"] = stream
    ws = P.Workspace(data, P.Settings(max_iters=100))
    lib, h = native.load(), ws._h
    native.check(lib.scs_begin(h, None, None, None), h)
    ms = native.C.c_double()
    native.check(lib.scs_bench_iters(h, 3, native.C.byref(ms)), h)
    native.check(lib.scs_bench_iters(h, 10, native.C.byref(ms)), h)
    fa = native.query(h, native.Q_FORMAT_A)
    del ws
    return ms.value * 1e3 / 10, fa


SHAPES = [("rows10_cols1e6", 2_000_000, 1_000_000, 21_000_000),
          ("rows20_cols1e5", 1_000_000, 100_000, 21_000_000),
          ("rows50_cols1e7", 400_000, 10_000_000, 21_000_000),
          ("rows5_cols4e6", 4_000_000, 4_000_000, 21_000_000)]
if "--crossover" in sys.argv:  # square shapes at ~400 / 800 / 1200 / 1700 entries per tile
    SHAPES = [(f"tile{e}", s, s, 21_000_000) for e, s in
              ((400, 940_000), (800, 660_000), (1200, 540_000), (1700, 455_000))]
if "--small" in sys.argv:  # dense tiles below the 2e7-nonzero gate
    SHAPES = [("nnz2.6e6", 125_000, 12_500, 2_700_000), ("nnz5.2e6", 250_000, 25_000, 5_300_000),
              ("nnz1e7", 500_000, 50_000, 10_500_000)]
for name, m, n, nz in SHAPES:
    d = problem(m, n, nz, 1)
    us1, f1 = timed(d, "1")
    us0, f0 = timed(d, "0")
    print(f"{name}: nnz={d.A.nnz} stream {us1:.1f} us/it (fmt {f1}), csr {us0:.1f} us/it (fmt {f0})", flush=True)
