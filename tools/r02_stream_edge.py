"""Streamed path (default heuristic: >= 2e7 nonzeros) on pathological
shapes: short-wide (a few rows of millions of entries), tall-thin, one dense
row + one dense column among sparse ones, empty rows/columns.  Compares
apply_a (A x, A^T y) with numpy bincount sums."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import native


def run(name, m, n, rows, cols, seed):
    rng = np.random.default_rng(seed)
    vals = rng.standard_normal(rows.size)
    order = np.lexsort((rows, cols))
    rows, cols, vals = rows[order], cols[order], vals[order]
    keep = np.ones(rows.size, bool)
    keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows.astype(np.int64), vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    t = time.time()
    ws = P.Workspace(data, P.Settings(normalize=False))
    q = (native.query(ws._h, native.Q_FORMAT_A), native.query(ws._h, native.Q_FORMAT_AT))
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    ax = np.bincount(rows, vals * x[cols], minlength=m)
    aty = np.bincount(cols, vals * y[rows], minlength=n)
    ga, gt = ws.apply_a(x), ws.apply_a(y, transpose=True)
    ea = np.abs(ga - ax).max() / (1 + np.abs(ax).max())
    et = np.abs(gt - aty).max() / (1 + np.abs(aty).max())
    ok = ea < 1e-12 and et < 1e-12
    print(f"{name}: m={m} n={n} nnz={rows.size} setup+apply {time.time() - t:.1f}s stream={q} errA={ea:.2e} errAt={et:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    rng = np.random.default_rng(0)
    res = []
    # short-wide: 8 rows x 3e6 columns, each row ~2.6e6 entries
    m, n, nz = 8, 3_000_000, 21_000_000
    res.append(run("short-wide", m, n, rng.integers(0, m, nz), rng.integers(0, n, nz), 1))
    # tall-thin: 2.1e7 rows x 6 columns
    m, n, nz = 21_000_000, 6, 21_000_000
    res.append(run("tall-thin", m, n, rng.integers(0, m, nz), rng.integers(0, n, nz), 2))
    # random sparse + one dense row + one dense column + empty rows / columns
    m, n, nz = 2_000_000, 1_000_000, 20_000_000
    r = rng.integers(0, m // 2, nz) * 2          # odd rows empty
    c = rng.integers(0, n // 2, nz) * 2          # odd columns empty
    r = np.concatenate([r, np.full(n // 2, 7), np.arange(0, m, 2)])
    c = np.concatenate([c, np.arange(0, n, 2), np.full(m // 2, 5)])
    res.append(run("dense-row-col", m, n, r, c, 3))
    print("ALL OK" if all(res) else "SOME FAILED")
    sys.exit(0 if all(res) else 1)


if __name__ == "__main__":
    main()
