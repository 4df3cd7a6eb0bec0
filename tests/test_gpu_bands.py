"""GPU tests of the row-banded A^T passes (setup_bands in csrc/solver.cu),
forced on for small problems with SCS_BANDS (read at Workspace creation).
The heuristic only bands A^T when its gathered vectors exceed the L2
(config 5), so without this the parity fixtures would not exercise it."""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import parallel

from _fixtures import load, rel

pytestmark = pytest.mark.gpu


def dense(colptr, rowidx, vals, m):
    n = colptr.size - 1
    A = np.zeros((m, n))
    A[rowidx, np.repeat(np.arange(n), np.diff(colptr))] = vals
    return A


@pytest.mark.parametrize("bands", [2, 5, 32])
@pytest.mark.parametrize("shape", [(40, 20, 0.3), (3000, 1000, 0.01), (200, 9000, 0.002),
                                   (9000, 200, 0.05)])
def test_banded_products_match_dense(monkeypatch, bands, shape):
    monkeypatch.setenv("SCS_BANDS", str(bands))
    m, n, dens = shape
    rng = np.random.default_rng(m + n + bands)
    lin = np.unique(rng.integers(0, m * n, max(1, int(dens * m * n))))
    cols, rows = np.divmod(lin, m)
    vals = rng.standard_normal(lin.size)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    ws = P.Workspace(data, P.Settings(normalize=False))
    A = dense(colptr, rows, vals, m)
    y = rng.standard_normal(m)
    tol = 1e-12 * (1 + np.abs(A).sum())
    np.testing.assert_allclose(ws.apply_a(y, transpose=True), A.T @ y, rtol=0, atol=tol)
    x = rng.standard_normal(n)
    np.testing.assert_allclose(ws.apply_a(x), A @ x, rtol=0, atol=tol)


@pytest.mark.parametrize("name", ["c1_lp_soc", "mixed", "ref_portfolio", "c2_lp_unbounded",
                                  "ref_lp_infeasible"])
def test_banded_golden_trajectories(monkeypatch, name):
    monkeypatch.setenv("SCS_BANDS", "4")
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


def test_banded_sharded_emulated(monkeypatch):
    """Bands inside each shard: band partials summed, then all-reduced."""
    prob = G.gen_lasso(300, 5000, 60000, seed=3)
    st = P.Settings(max_iters=60)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    ref = {}
    sol1 = P.Workspace(data, st).solve(on_iteration=lambda s: ref.__setitem__(s.iter, s.u.copy()))
    monkeypatch.setenv("SCS_BANDS", "3")
    n = colptr.size - 1
    parts = {}
    res = parallel.emulated_solve(prob, st, 2, on_iteration=lambda r, s: parts.setdefault(
        s.iter, {}).__setitem__(r, s.u.copy()))
    for k, by in parts.items():
        u = np.concatenate([by[0][:n], by[0][n:-1], by[1][n:-1], by[0][-1:]])
        assert rel(u, ref[k]) < 1e-9, k
    assert all(s.status == sol1.status for _, s in res)


def test_banded_deterministic(monkeypatch):
    monkeypatch.setenv("SCS_BANDS", "5")
    prob = G.gen_lasso(300, 5000, 60000, seed=4)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    runs = [P.Workspace(data, P.Settings(max_iters=40)).solve() for _ in range(2)]
    assert np.array_equal(runs[0].x, runs[1].x) and np.array_equal(runs[0].y, runs[1].y)


# ---- long rows split into pieces (setup_split), forced with SCS_SPLIT=1 ----

@pytest.mark.parametrize("shape", [(40, 20, 0.3), (3000, 1000, 0.01), (200, 9000, 0.002),
                                   (9000, 200, 0.05)])
def test_split_products_match_dense(monkeypatch, shape):
    monkeypatch.setenv("SCS_SPLIT", "1")
    m, n, dens = shape
    rng = np.random.default_rng(m * 3 + n)
    lin = np.unique(rng.integers(0, m * n, max(1, int(dens * m * n))))
    # plus one dense row and one dense column (the skew the split targets)
    lin = np.unique(np.concatenate([lin, np.arange(n) * m + 1, 2 * m + np.arange(m)]))
    cols, rows = np.divmod(lin, m)
    vals = rng.standard_normal(lin.size)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    ws = P.Workspace(data, P.Settings(normalize=False))
    A = dense(colptr, rows, vals, m)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    tol = 1e-12 * (1 + np.abs(A).sum())
    np.testing.assert_allclose(ws.apply_a(x), A @ x, rtol=0, atol=tol)
    np.testing.assert_allclose(ws.apply_a(y, transpose=True), A.T @ y, rtol=0, atol=tol)


@pytest.mark.parametrize("name", ["c1_lp_soc", "mixed", "ref_portfolio", "ref_lp_infeasible",
                                  "c2_lp_unbounded"])
def test_split_golden_trajectories(monkeypatch, name):
    monkeypatch.setenv("SCS_SPLIT", "1")
    _golden(name)


def _golden(name):
    d = load(name)
    st = d["settings"]
    settings = P.Settings(alpha=st["alpha"], max_iters=st["max_iters"], eps_pri=st["eps_pri"],
                          eps_dual=st["eps_dual"], eps_gap=st["eps_gap"],
                          eps_infeas=st["eps_infeas"], eps_unbdd=st["eps_unbdd"],
                          check_interval=st["check_interval"], cg_max=st["cg_max"],
                          cg_tol=st["cg_tol"], normalize=st["normalize"], sweeps=st["sweeps"])
    data = P.ProblemData(P.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"]),
                         d["b"], d["c"], P.ConeSpec.from_any(d["cone"]))
    kept = [int(k) for k in d["kept"]]
    got = {}
    sol = P.Workspace(data, settings).solve(
        on_iteration=lambda s: got.__setitem__(s.iter, s.u.copy()) if s.iter in kept else None)
    for i, k in enumerate(kept):
        assert rel(got[k], d["us"][i]) < 1e-9, (name, k)
    assert sol.status.value == d["status"]
    assert abs(sol.info.iterations - d["iterations"]) <= max(2, d["iterations"] // 200)


def test_split_sharded_emulated(monkeypatch):
    prob = G.gen_portfolio_c4(300, 5, 30, seed=2)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    st = P.Settings(max_iters=40)
    ref = {}
    P.Workspace(data, st).solve(on_iteration=lambda s: ref.__setitem__(s.iter, s.u.copy()))
    monkeypatch.setenv("SCS_SPLIT", "1")
    n = colptr.size - 1
    parts = {}
    parallel.emulated_solve(prob, st, 2, on_iteration=lambda r, s: parts.setdefault(
        s.iter, {}).__setitem__(r, s.u.copy()))
    for k, by in parts.items():
        u = np.concatenate([by[0][:n], by[0][n:-1], by[1][n:-1], by[0][-1:]])
        assert rel(u, ref[k]) < 1e-9, k
