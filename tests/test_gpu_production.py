"""Parity at the benchmarked scale (BASELINE configs 3 and 5), through the
production SpMV format (TMA-streamed tiles, chosen automatically from 4e6
nonzeros) with no SCS_STREAM_* overrides.

* Config 3 (1e8 nonzeros) against conesplit itself: the fixture
  tests/golden/c3_ref.npz was produced by running the reference's
  Workspace.solve (solver.py:336-378) for 50 iterations on the same instance
  (tests/golden/make_c3_golden.py; the instance is bit-identical between
  the native generator used here and the numpy twin used there,
  tests/test_generators.py).  Checked: equilibration (D, E samples, sigma,
  rho) to 1e-12; ||u||, ||v|| after every iteration and 2e4 sampled entries
  at k = 1, 2, 5, 10, 20, 50 to the north star's 1e-9; the cumulative CG
  count after every iteration exactly (embedding.py:112); every termination
  check's eight Residuals values (scaling.py:148-207) in the default
  residual-recurrence mode; the final status (max_iters_reached, the
  post-loop rule of solver.py:364-369) and iteration count exactly.
* Config 5 (1e9 nonzeros): the reference cannot run it in host RAM, so the
  streamed path is checked against the CSR kernel path (SCS_STREAM=0) on the
  same instance -- the first 50 iterates to 1e-12, identical CG counts.
"""

import math
import os

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import native
from paper_1312_3039_b200.api import _STATUS_BY_CODE

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
C3 = dict(p=50_000, q=899_998, nnz=100_000_000, seed=1)   # bench.py CONFIGS["c3"]
C5 = dict(p=500_000, q=8_999_998, nnz=1_000_000_000, seed=1)
ITERATE_TOL = 1e-9


def _data(cfg):
    colptr, rowidx, vals, b, c, cone = native.gen_lasso(
        cfg["p"], cfg["q"], cfg["nnz"] - 4 * cfg["p"] - 2, seed=cfg["seed"])
    m, n = b.size, colptr.size - 1
    A = object.__new__(P.SparseMatrix)  # generator output: skip the O(nnz) host validation
    A.nrows, A.ncols, A.colptr, A.rowidx, A.vals = m, n, colptr, rowidx, vals
    d = object.__new__(P.ProblemData)
    d.A, d.b, d.c, d.spec = A, b, c, P.ConeSpec.from_any(cone)
    return d


def _trajectory(ws, iters, snap, idx):
    """Step one iteration at a time through the C-ABI; per iteration: norms,
    cumulative CG count, and the Residuals of the check that completed in
    this step (the check of iteration k rides on step k + 1)."""
    lib, h = native.load(), ws._h
    native.check(lib.scs_begin(h, None, None, None), h)
    info = native.Info()
    out = dict(unorm=[], vnorm=[], cg=[], res=[], snap={})
    for k in range(1, iters + 1):
        native.check(lib.scs_step(h, 1, native.C.byref(info)), h)
        if info.iterations != k:
            break
        u, v = ws.state()
        out["unorm"].append(np.linalg.norm(u))
        out["vnorm"].append(np.linalg.norm(v))
        out["cg"].append(int(info.cg_iters))
        out["res"].append([float(x) for x in info.res])
        if k in snap:
            out["snap"][k] = (u[idx].copy(), v[idx].copy())
        if info.status >= 0:
            break
    native.check(lib.scs_finish(h, native.C.byref(info)), h)
    out["status"] = int(info.status)
    out["iterations"] = int(info.iterations)
    out["final_res"] = [float(x) for x in info.res]
    out["cg_total"] = int(info.cg_iters)
    return out


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _res_close(got, ref, tol):
    """Residuals: inf where the reference has inf (sign conditions), else
    relative agreement (the gap can cross zero: compared against its
    threshold scale, gap_thresh)."""
    for i, (g, r) in enumerate(zip(got, ref)):
        if math.isinf(r):
            assert math.isinf(g), (i, g, r)
            continue
        scale = abs(ref[5]) if i == 2 else abs(r)
        assert abs(g - r) <= tol * max(scale, 1e-300), (i, g, r)


@pytest.fixture(scope="module")
def c3_ref():
    return np.load(os.path.join(HERE, "golden", "c3_ref.npz"))


def test_c3_reference_parity(c3_ref):
    d = c3_ref
    data = _data(C3)
    assert data.A.rowidx.size == int(d["nnz"]) and data.m == int(d["m"])
    it = int(d["iterations"])
    ws = P.Workspace(data, P.Settings(max_iters=it, eps_pri=1e-3, eps_dual=1e-3, eps_gap=1e-3))
    h = ws._h
    # the production format ran: streamed tiles for A and A^T, default knobs
    assert not any(k.startswith("SCS_STREAM") for k in os.environ)
    assert native.query(h, native.Q_FORMAT_A) == 1 and native.query(h, native.Q_FORMAT_AT) == 1
    sc = ws.scal
    assert _rel(sc.D[d["didx"]], d["D"]) < 1e-12 and _rel(sc.E[d["eidx"]], d["E"]) < 1e-12
    assert math.isclose(sc.sigma, float(d["sigma"]), rel_tol=1e-12)
    assert math.isclose(sc.rho, float(d["rho"]), rel_tol=1e-12)
    snap = [int(k) for k in d["kept"]]
    t = _trajectory(ws, it, snap, d["idx"])
    assert len(t["unorm"]) == it
    for k in range(it):
        assert abs(t["unorm"][k] - d["unorm"][k]) <= ITERATE_TOL * d["unorm"][k], k
        assert abs(t["vnorm"][k] - d["vnorm"][k]) <= ITERATE_TOL * d["vnorm"][k], k
    for i, k in enumerate(snap):
        assert _rel(t["snap"][k][0], d["us"][i]) < ITERATE_TOL, k
        assert _rel(t["snap"][k][1], d["vs"][i]) < ITERATE_TOL, k
    # cumulative CG count (incl. the setup solve of g) after every iteration
    np.testing.assert_array_equal(t["cg"], d["cg_total"][:it])
    assert t["cg_total"] == int(d["cg_iters"])
    # residuals of every check: the check of iteration k completes in step k + 1
    for k in range(1, it):
        _res_close(t["res"][k], d["res"][k - 1], 1e-7)
    _res_close(t["final_res"], d["final_res"], 1e-7)
    assert _STATUS_BY_CODE[t["status"]].value == str(d["status"])  # max_iters_reached
    assert t["iterations"] == it


def test_c5_streamed_matches_csr():
    data = _data(C5)
    ell = data.n + data.m + 1
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(ell, 100_000, replace=False))
    snap = (1, 2, 5, 10, 20, 50)
    st = P.Settings(max_iters=50, eps_pri=1e-3, eps_dual=1e-3, eps_gap=1e-3)
    ws = P.Workspace(data, st)
    assert native.query(ws._h, native.Q_FORMAT_A) == 1
    assert native.query(ws._h, native.Q_FORMAT_AT) == 1
    ts = _trajectory(ws, 50, snap, idx)
    del ws
    os.environ["SCS_STREAM"] = "0"
    try:
        wc = P.Workspace(data, st)
    finally:
        del os.environ["SCS_STREAM"]
    assert native.query(wc._h, native.Q_FORMAT_A) == 0
    tc = _trajectory(wc, 50, snap, idx)
    del wc
    assert len(ts["unorm"]) == len(tc["unorm"]) == 50
    for k in range(50):
        assert abs(ts["unorm"][k] - tc["unorm"][k]) <= 1e-12 * tc["unorm"][k], k
        assert abs(ts["vnorm"][k] - tc["vnorm"][k]) <= 1e-12 * tc["vnorm"][k], k
    for k in snap:
        assert _rel(ts["snap"][k][0], tc["snap"][k][0]) < 1e-12, k
        assert _rel(ts["snap"][k][1], tc["snap"][k][1]) < 1e-12, k
    assert ts["cg"] == tc["cg"]
    assert ts["status"] == tc["status"] and ts["iterations"] == tc["iterations"]


def test_mid_size_default_streamed_matches_csr():
    """The mid-size regime the r02 gate now streams (1e7 nonzeros, ~600
    dense tiles): default format against the CSR kernel, 30 iterates."""
    data = _data(dict(p=15_000, q=270_000, nnz=10_000_000, seed=3))
    ell = data.n + data.m + 1
    idx = np.sort(np.random.default_rng(6).choice(ell, 20_000, replace=False))
    snap = (1, 5, 30)
    st = P.Settings(max_iters=30, eps_pri=1e-3, eps_dual=1e-3, eps_gap=1e-3)
    ws = P.Workspace(data, st)
    assert native.query(ws._h, native.Q_FORMAT_A) == 1
    assert native.query(ws._h, native.Q_FORMAT_AT) == 1
    ts = _trajectory(ws, 30, snap, idx)
    del ws
    os.environ["SCS_STREAM"] = "0"
    try:
        wc = P.Workspace(data, st)
    finally:
        del os.environ["SCS_STREAM"]
    tc = _trajectory(wc, 30, snap, idx)
    del wc
    for k in range(len(tc["unorm"])):
        assert abs(ts["unorm"][k] - tc["unorm"][k]) <= 1e-12 * tc["unorm"][k], k
        assert abs(ts["vnorm"][k] - tc["vnorm"][k]) <= 1e-12 * tc["vnorm"][k], k
    for k in snap:
        assert _rel(ts["snap"][k][0], tc["snap"][k][0]) < 1e-12, k
    assert ts["cg"] == tc["cg"]
    assert ts["status"] == tc["status"] and ts["iterations"] == tc["iterations"]
