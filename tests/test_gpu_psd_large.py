"""GPU parity of the cooperative-grid Jacobi for large PSD blocks
(`k_psd_grid`, sides beyond the shared-memory side; the
RPCA block of generators.py:197-286).

The PSD projection is unique, so at these sides numpy's eigh (the pure-Python
Jacobi restatement is too slow) and the r01 one-CTA path (SCS_PSD_GRID=0,
itself checked against eigh) are the checkers.  The reference's stopping
rule (_kernels.py:137-191) is kept, so results agree to rounding.
"""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import native
from oracle import scs_oracle as O

from _fixtures import rel

pytestmark = pytest.mark.gpu


def _eigh_proj(x, k):
    m = O.svec_to_mat(x, k)
    w, v = np.linalg.eigh(0.5 * (m + m.T))
    return O.mat_to_svec((v * np.maximum(w, 0.0)) @ v.T)


@pytest.mark.parametrize("sides", [[130], [1000], [2000, 3, 501], [117, 116, 20, 300]])
def test_grid_psd_vs_eigh(sides):
    rng = np.random.default_rng(7 + sum(sides))
    cone = {"s": sides}
    x = rng.standard_normal(O.cone_from_spec(cone).dim)
    got = native.project_cone(x, cone, "dual")
    off = 0
    for k in sides:
        d = k * (k + 1) // 2
        exp = _eigh_proj(x[off:off + d], k)
        np.testing.assert_allclose(got[off:off + d], exp, atol=1e-9 * (1 + np.abs(x).max()))
        off += d


def test_grid_psd_low_rank_and_clustered():
    """Clustered spectra (many equal eigenvalues: the tiny-entry rule) and a
    rank-deficient input, primal and dual projections."""
    rng = np.random.default_rng(3)
    k = 400
    q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    w = np.concatenate([np.full(150, 2.0), np.full(150, -1.0), rng.standard_normal(100)])
    m = (q * w) @ q.T
    x = O.mat_to_svec(m)
    for kind in ("dual", "primal"):
        got = native.project_cone(x, {"s": [k]}, kind)
        exp = _eigh_proj(x, k) if kind == "dual" else x + _eigh_proj(-x, k)
        np.testing.assert_allclose(got, exp, atol=1e-9 * (1 + np.abs(x).max()))


def test_grid_matches_cta_path(monkeypatch):
    rng = np.random.default_rng(11)
    cone = {"l": 5, "q": [4], "s": [200, 9, 160]}
    x = rng.standard_normal(O.cone_from_spec(cone).dim)
    got = native.project_cone(x, cone, "dual")
    monkeypatch.setenv("SCS_PSD_GRID", "0")
    old = native.project_cone(x, cone, "dual")
    np.testing.assert_allclose(got, old, atol=1e-10 * (1 + np.abs(x).max()))


def _min_eig_sdp(k, seed):
    """min tr(C X) s.t. tr(X) = 1, X PSD (optimum: lambda_min(C)), in the
    reference's standard form: one zero-cone row, then s = x in the PSD cone."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((k, k))
    C = 0.5 * (g + g.T) / np.sqrt(k)
    d = k * (k + 1) // 2
    diag = O.mat_to_svec(np.eye(k))
    dense = np.zeros((1 + d, d))
    dense[0] = diag
    dense[1:] = -np.eye(d)
    b = np.zeros(1 + d)
    b[0] = 1.0
    c = O.mat_to_svec(C)
    colptr, rowidx, vals = [0], [], []
    for j in range(d):
        nz = np.nonzero(dense[:, j])[0]
        rowidx.extend(nz)
        vals.extend(dense[nz, j])
        colptr.append(len(rowidx))
    A = P.SparseMatrix(1 + d, d, np.array(colptr, np.int64), np.array(rowidx, np.int64),
                       np.array(vals, np.float64))
    return P.ProblemData(A, b, c, P.ConeSpec.from_any({"z": 1, "s": [k]})), C


def test_sdp_solve_grid_vs_cta_path(monkeypatch):
    """Solves through the graph-captured iteration (the cooperative launch
    inside the CUDA graph): the first 50 iterates equal the one-CTA path's to
    1e-9; the full solve reaches lambda_min(C)."""
    prob, C = _min_eig_sdp(150, 5)

    def traj():
        t = {}
        P.Workspace(prob, P.Settings(max_iters=50)).solve(
            on_iteration=lambda s: t.__setitem__(s.iter, s.u.copy()))
        return t

    got = traj()
    monkeypatch.setenv("SCS_PSD_GRID", "0")
    old = traj()
    monkeypatch.delenv("SCS_PSD_GRID")
    assert len(old) == 50
    for it in old:
        assert rel(got[it], old[it]) < 1e-9, it
    sol = P.solve(prob, P.Settings(eps_pri=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=5000))
    assert sol.status is P.Status.SOLVED
    lam = np.linalg.eigvalsh(C)[0]
    assert abs(sol.objective - lam) <= 1e-2 * (1 + abs(lam))


def _tuple(prob):
    A = prob.A
    sp = prob.spec
    return (A.colptr, A.rowidx, A.vals, prob.b, prob.c,
            {"z": sp.zero_dim, "l": sp.nonneg_dim, "q": list(sp.soc_dims), "s": list(sp.psd_sides)})


def test_sdp_sharded_paths_match_single():
    """Row-sharded code paths with a large PSD block: the NCCL communicator
    (one rank, sharded path forced on: the cooperative launch captured in one
    graph with the all-reduces, and the device extraction's all-reduced b'y),
    and the emulated 2-shard group (which keeps one CTA per block)."""
    from paper_1312_3039_b200 import parallel
    prob, _ = _min_eig_sdp(130, 9)
    st = P.Settings(max_iters=60)
    t1 = {}
    sol1 = P.Workspace(prob, st).solve(
        on_iteration=lambda s: t1.__setitem__(s.iter, s.u.copy()))
    lib = native.load()
    buf = (native.C.c_uint8 * 128)()
    native.check(lib.scs_nccl_unique_id(buf))
    colptr, rowidx, vals, b, c, cone = _tuple(prob)
    m = b.size
    spec = parallel.ShardSpec(0, 1, np.array([0, m], np.int64), nccl_id=bytes(buf), force=True)
    shard = parallel.shard_problem(colptr, rowidx, vals, b, c, cone, spec.bounds, 0)
    ws = P.Workspace(shard, st, dist=spec)
    t2 = {}
    ws.solve(on_iteration=lambda s: t2.__setitem__(s.iter, s.u.copy()))
    for k in t1:
        assert rel(t2[k], t1[k]) < 1e-9, k
    sol2 = ws.solve()  # graph-launched loop
    assert sol2.status == sol1.status and sol2.info.iterations == sol1.info.iterations
    assert abs(sol2.objective - sol1.objective) <= 1e-9 * (1 + abs(sol1.objective))
    res = parallel.emulated_solve(_tuple(prob), st, 2, bounds=np.array([0, 1, m], np.int64))
    for _, s in res:
        assert s.status == sol1.status and s.info.iterations == sol1.info.iterations


def test_two_workspaces_different_psd_smem():
    """Two live workspaces on one GPU whose PSD blocks need different dynamic
    shared memory (sides 100 and 60: 160 KB and 58 KB in k_cone_apply): the
    per-device kernel attribute is raised once and never lowered, so the
    first workspace still solves after the second one's setup, and each
    equals a solve alone."""
    big, _ = _min_eig_sdp(100, 21)
    small, _ = _min_eig_sdp(60, 22)
    st = P.Settings(max_iters=40)
    alone_big = P.Workspace(big, st).solve()
    alone_small = P.Workspace(small, st).solve()
    wa = P.Workspace(big, st)
    wb = P.Workspace(small, st)
    ra = wa.solve()
    rb = wb.solve()
    ra2 = wa.solve()
    assert np.array_equal(ra.x, alone_big.x) and np.array_equal(ra2.x, alone_big.x)
    assert np.array_equal(rb.x, alone_small.x)
