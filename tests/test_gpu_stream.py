"""GPU tests of the TMA-streamed tile SpMV (csrc/stream.cuh), forced on for
small problems (SCS_STREAM=1 is read at Workspace creation; the size
heuristic only enables it from 4e6 nonzeros and dense tiles).  The knobs shrink the format
so that small matrices exercise every path: many slabs (SCS_STREAM_W),
tiles cut into several pieces (SCS_STREAM_CAP), slab-range splits with the
combine kernel (SCS_STREAM_SPLITS), and CSR units for sparse sub-blocks
(SCS_STREAM_MIN)."""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G

from _fixtures import load, rel

pytestmark = pytest.mark.gpu

VARIANTS = {
    "default": {},
    "narrow": {"SCS_STREAM_W": "64"},
    "pieces": {"SCS_STREAM_W": "512", "SCS_STREAM_CAP": "6208"},
    "splits": {"SCS_STREAM_W": "128", "SCS_STREAM_SPLITS": "3"},
    "splits9": {"SCS_STREAM_W": "64", "SCS_STREAM_SPLITS": "11"},
    "csr": {"SCS_STREAM_MIN": "1000000000"},
    "mixed": {"SCS_STREAM_W": "256", "SCS_STREAM_MIN": "300", "SCS_STREAM_SPLITS": "2"},
}


@pytest.fixture(params=sorted(VARIANTS))
def stream(request, monkeypatch):
    monkeypatch.setenv("SCS_STREAM", "1")
    for k, v in VARIANTS[request.param].items():
        monkeypatch.setenv(k, v)
    return request.param


def dense(colptr, rowidx, vals, m):
    n = colptr.size - 1
    A = np.zeros((m, n))
    A[rowidx, np.repeat(np.arange(n), np.diff(colptr))] = vals
    return A


def random_csc(m, n, dens, seed):
    rng = np.random.default_rng(seed)
    nnz = max(1, int(dens * m * n))
    lin = np.unique(rng.integers(0, m * n, nnz))
    cols, rows = np.divmod(lin, m)
    vals = rng.standard_normal(lin.size)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    return colptr, rows, vals


@pytest.mark.parametrize("shape", [(40, 20, 0.3), (3000, 1000, 0.01), (200, 9000, 0.002),
                                   (9000, 200, 0.05), (13000, 5000, 0.0008)])
def test_stream_products_match_dense(stream, shape):
    """Random sparsity: rows longer than a slab, empty rows and columns,
    several sub-blocks (pair units, a partial last sub-block)."""
    m, n, dens = shape
    colptr, rows, vals = random_csc(m, n, dens, m + n)
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    ws = P.Workspace(data, P.Settings(normalize=False))
    A = dense(colptr, rows, vals, m)
    rng = np.random.default_rng(7)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    tol = 1e-12 * (1 + np.abs(A).sum())
    np.testing.assert_allclose(ws.apply_a(x), A @ x, rtol=0, atol=tol)
    np.testing.assert_allclose(ws.apply_a(y, transpose=True), A.T @ y, rtol=0, atol=tol)


def test_stream_skewed_rows(stream):
    """A dense row and a dense column among short ones (pinned depths far
    above E / 32: deeper sections, narrower slabs or a CSR unit)."""
    m, n = 9000, 6000
    colptr, rows, vals = random_csc(m, n, 0.0005, 11)
    A = dense(colptr, rows, vals, m)
    A[17, :] = np.linspace(-1, 1, n)
    A[:, 4321] = np.linspace(2, 3, m)
    cols, rws = np.nonzero(A.T)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rws, A.T[cols, rws]), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    ws = P.Workspace(data, P.Settings(normalize=False))
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    tol = 1e-12 * (1 + np.abs(A).sum())
    np.testing.assert_allclose(ws.apply_a(x), A @ x, rtol=0, atol=tol)
    np.testing.assert_allclose(ws.apply_a(y, transpose=True), A.T @ y, rtol=0, atol=tol)


@pytest.mark.parametrize("name", ["c1_lp_soc", "mixed", "ref_portfolio", "c2_lp_unbounded",
                                  "c2_lp_infeasible"])
def test_stream_golden_trajectories(stream, name):
    """Every pass of the iteration (NV = 1 and 2, strides 1 and 2, fused
    epilogues and split partials) against the reference's iterates."""
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
    assert sol.info.iterations == d["iterations"]


def test_stream_lasso_deterministic(monkeypatch):
    """Same inputs, same bits: the streamed accumulation order is fixed."""
    monkeypatch.setenv("SCS_STREAM", "1")
    monkeypatch.setenv("SCS_STREAM_W", "256")
    prob = G.gen_lasso(300, 5000, 60000, seed=3)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    runs = [P.Workspace(data, P.Settings(max_iters=40)).solve() for _ in range(2)]
    assert np.array_equal(runs[0].x, runs[1].x) and np.array_equal(runs[0].y, runs[1].y)


@pytest.mark.parametrize("name", ["c1_lp_soc", "c2_lp_infeasible", "ref_lasso"])
@pytest.mark.parametrize("world", [2, 3])
def test_stream_row_shards_match_reference(monkeypatch, name, world):
    """Row shards (emulated all-reduce group) over streamed tiles: raw
    partial products of the A^T passes (EpiRaw through the streamed kernel,
    split partials), all-reduced, against the reference's first iterates."""
    from test_gpu_sharded import fixture_prob, settings_from, sharded
    monkeypatch.setenv("SCS_STREAM", "1")
    monkeypatch.setenv("SCS_STREAM_W", "256")
    prob, d = fixture_prob(name)
    st = settings_from(d["settings"])
    res, traj = sharded(prob, st, world)
    kept = [int(k) for k in d["kept"]]
    for i, k in enumerate(kept):
        if k in traj:
            assert rel(traj[k], d["us"][i]) < 1e-9, (name, world, k)
    assert all(s.status.value == d["status"] for _, s in res)


def _unique_coo(m, n, nz, seed):
    rng = np.random.default_rng(seed)
    key = np.unique(rng.integers(0, n, nz).astype(np.int64) * m + rng.integers(0, m, nz))
    cols, rows = np.divmod(key, m)
    return rows, cols, rng.standard_normal(key.size)


@pytest.mark.parametrize("name,m,n,nz,streamed", [
    ("dense_tiles", 1_000_000, 100_000, 21_000_000, 1),     # ~3400 entries per tile
    ("sparse_tiles", 2_000_000, 1_000_000, 21_000_000, 0),  # ~175 entries per tile: CSR kernel
    ("short_wide", 16, 4_000_000, 25_000_000, 1),           # 16 rows of ~1.4e6 entries
    ("tall_thin", 30_000_000, 6, 24_000_000, 1),            # 6 columns of ~4e6 entries
    ("mid_dense", 500_000, 50_000, 10_500_000, 1),          # 1.05e7 nonzeros, ~6500 per tile
    ("small", 125_000, 12_500, 2_700_000, 0),               # below 4e6 nonzeros: CSR kernel
    ("few_tiles", 100_000, 10_000, 10_000_000, 0),          # dense, but 25 x 3 tiles: CSR kernel
])
def test_default_format_by_tile_density(name, m, n, nz, streamed):
    """Production heuristic (no SCS_STREAM knob): >= 4e6 nonzeros streams a
    matrix only when its average tile holds >= 1000 entries and it has at
    least 2 tiles per SM (sparser tiles
    ran 2-3x slower than the CSR kernel); extreme row / column lengths go
    through the dense-section handling.  Products against numpy sums."""
    rows, cols, vals = _unique_coo(m, n, nz, 5)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    data = P.ProblemData(P.SparseMatrix(m, n, colptr, rows, vals), np.ones(m), np.ones(n),
                         P.ConeSpec(nonneg_dim=m))
    ws = P.Workspace(data, P.Settings(normalize=False))
    from paper_1312_3039_b200 import native
    assert native.query(ws._h, native.Q_FORMAT_A) == streamed
    assert native.query(ws._h, native.Q_FORMAT_AT) == streamed
    rng = np.random.default_rng(9)
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    ax = np.bincount(rows, vals * x[cols], minlength=m)
    aty = np.bincount(cols, vals * y[rows], minlength=n)
    assert np.abs(ws.apply_a(x) - ax).max() <= 1e-12 * (1 + np.abs(ax).max())
    assert np.abs(ws.apply_a(y, transpose=True) - aty).max() <= 1e-12 * (1 + np.abs(aty).max())
