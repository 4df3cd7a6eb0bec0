"""GPU tests of the slab-tiled SpMV (csrc/tiled.cuh), forced on for small
problems (SCS_TILED=1 is read at Workspace creation).  The size heuristic
only enables it for large matrices, so without this the small parity
fixtures would exercise the CSR kernel alone."""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import parallel

from _fixtures import load, rel

pytestmark = pytest.mark.gpu


@pytest.fixture
def tiled(monkeypatch):
    monkeypatch.setenv("SCS_TILED", "1")


def dense(colptr, rowidx, vals, m):
    n = colptr.size - 1
    A = np.zeros((m, n))
    A[rowidx, np.repeat(np.arange(n), np.diff(colptr))] = vals
    return A


@pytest.mark.parametrize("shape", [(40, 20, 0.3), (3000, 1000, 0.01), (200, 9000, 0.002),
                                   (9000, 200, 0.05), (5000, 5000, 0.0008)])
def test_tiled_products_match_dense(tiled, shape):
    """Random sparsity incl. rows that span many warps, empty rows/columns,
    several slabs (cols > 4096) and row blocks."""
    m, n, dens = shape
    rng = np.random.default_rng(m + n)
    nnz = max(1, int(dens * m * n))
    lin = np.unique(rng.integers(0, m * n, nnz))
    cols, rows = np.divmod(lin, m)
    vals = rng.standard_normal(lin.size)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    ws = P.Workspace(data, P.Settings(normalize=False))
    A = dense(colptr, rows, vals, m)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    np.testing.assert_allclose(ws.apply_a(x), A @ x, rtol=0, atol=1e-12 * (1 + np.abs(A).sum()))
    np.testing.assert_allclose(ws.apply_a(y, transpose=True), A.T @ y, rtol=0,
                               atol=1e-12 * (1 + np.abs(A).sum()))


def test_tiled_row_slices(tiled):
    """Row slices of an LP (the shapes that exposed a boundary-merge race)."""
    d = load("ref_lp_infeasible")
    colptr, rowidx, vals, b, c = d["colptr"], d["rowidx"], d["vals"], d["b"], d["c"]
    n = colptr.size - 1
    for lo, hi in ((0, 21), (21, 40), (14, 27), (0, 40)):
        cp, ri, va = parallel.slice_rows(colptr, rowidx, vals, lo, hi)
        mk = hi - lo
        data = P.ProblemData(P.SparseMatrix(mk, n, cp, ri, va), b[lo:hi], c,
                             P.ConeSpec(nonneg_dim=mk))
        ws = P.Workspace(data, P.Settings(normalize=False))
        x = np.arange(n) + 1.0
        np.testing.assert_allclose(ws.apply_a(x), dense(cp, ri, va, mk) @ x, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["c1_lp_soc", "mixed", "ref_portfolio", "c2_lp_unbounded"])
def test_tiled_golden_trajectories(tiled, name):
    d = load(name)
    st = d["settings"]
    settings = P.Settings(alpha=st["alpha"], max_iters=st["max_iters"], eps_pri=st["eps_pri"],
                          eps_dual=st["eps_dual"], eps_gap=st["eps_gap"],
                          eps_infeas=st["eps_infeas"], eps_unbdd=st["eps_unbdd"],
                          check_interval=st["check_interval"], cg_max=st["cg_max"],
                          cg_tol=st["cg_tol"], normalize=st["normalize"], sweeps=st["sweeps"])
    data = P.ProblemData(P.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"]),
                         d["b"], d["c"], P.ConeSpec.from_any(d["cone"]))
    ws = P.Workspace(data, settings)
    kept = [int(k) for k in d["kept"]]
    got = {}
    sol = ws.solve(on_iteration=lambda s: got.__setitem__(s.iter, s.u.copy())
                   if s.iter in kept else None)
    for i, k in enumerate(kept):
        assert rel(got[k], d["us"][i]) < 1e-9, (name, k)
    assert sol.status.value == d["status"]
    assert abs(sol.info.iterations - d["iterations"]) <= max(2, d["iterations"] // 200)


def test_tiled_lasso_deterministic(tiled):
    """Same inputs, same bits: the tiled reduction order is fixed."""
    prob = G.gen_lasso(300, 5000, 60000, seed=3)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    runs = [P.Workspace(data, P.Settings(max_iters=40)).solve() for _ in range(2)]
    assert np.array_equal(runs[0].x, runs[1].x) and np.array_equal(runs[0].y, runs[1].y)
