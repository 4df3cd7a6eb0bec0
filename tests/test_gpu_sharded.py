"""GPU tests of the row-sharded path on one GPU.

The shards run as host threads joined by the in-process emulated all-reduce
group (the same kernels and all-reduce points as the NCCL build; no kernel
waits on another shard), and -- for the NCCL code itself -- a one-rank NCCL
communicator with the sharded code path forced on.  Each must reproduce
the single-GPU (= reference-parity) trajectory to 1e-9 and its status.
"""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import native, parallel

from _fixtures import load, rel

pytestmark = pytest.mark.gpu

TOL = 1e-9


def fixture_prob(name):
    d = load(name)
    return (d["colptr"], d["rowidx"], d["vals"], d["b"], d["c"], d["cone"]), d


def settings_from(st, **over):
    kw = dict(alpha=st["alpha"], max_iters=st["max_iters"], eps_pri=st["eps_pri"],
              eps_dual=st["eps_dual"], eps_gap=st["eps_gap"], eps_infeas=st["eps_infeas"],
              eps_unbdd=st["eps_unbdd"], check_interval=st["check_interval"],
              cg_max=st["cg_max"], cg_tol=st["cg_tol"], normalize=st["normalize"],
              sweeps=st["sweeps"])
    kw.update(over)
    return P.Settings(**kw)


def single(prob, st, upto=50):
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    traj = {}
    ws = P.Workspace(data, st)
    sol = ws.solve(on_iteration=lambda s: traj.__setitem__(s.iter, s.u.copy())
                   if s.iter <= upto else None)
    return ws, sol, traj


def sharded(prob, st, world, bounds=None, upto=50):
    parts = {}

    def cb(rank, s):
        if s.iter <= upto:
            parts.setdefault(s.iter, {})[rank] = s.u.copy()

    res = parallel.emulated_solve(prob, st, world, bounds=bounds, on_iteration=cb)
    n = prob[0].size - 1
    traj = {}
    for k, by_rank in parts.items():
        if len(by_rank) == world:
            u0 = by_rank[0]
            y = np.concatenate([by_rank[r][n:-1] for r in range(world)])
            traj[k] = np.concatenate([u0[:n], y, u0[-1:]])
            for r in range(1, world):  # x-part and tau are replicated bit-for-bit
                assert np.array_equal(by_rank[r][:n], u0[:n])
                assert by_rank[r][-1] == u0[-1]
    return res, traj


CASES = ["c1_lp_soc", "mixed", "ref_portfolio", "ref_lp_infeasible", "ref_lasso", "ref_rpca"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("world", [2, 3])
def test_emulated_shards_match_single_gpu(name, world):
    prob, d = fixture_prob(name)
    st = settings_from(d["settings"])
    ws1, sol1, traj1 = single(prob, st)
    res, trajk = sharded(prob, st, world)
    for k in sorted(traj1):
        assert rel(trajk[k], traj1[k]) < TOL, (name, world, k, rel(trajk[k], traj1[k]))
    sols = [s for _, s in res]
    assert all(s.status == sol1.status for s in sols)
    assert all(s.info.iterations == sol1.info.iterations for s in sols)
    if sol1.status in (P.Status.SOLVED, P.Status.MAX_ITERS_REACHED):
        assert abs(sols[0].primal_obj - sol1.primal_obj) <= 1e-9 * max(1, abs(sol1.primal_obj))
        assert abs(sols[0].dual_obj - sol1.dual_obj) <= 1e-9 * max(1, abs(sol1.dual_obj))
        y = parallel.gather_vector([s.y for s in sols])
        assert rel(y, sol1.y) < 1e-8
        assert abs(sols[0].info.pri_res - sol1.info.pri_res) <= 1e-9 + 1e-6 * sol1.info.pri_res
    elif sol1.certificate is not None and sol1.status is P.Status.INFEASIBLE:
        cert = parallel.gather_vector([s.certificate for s in sols])
        assert rel(cert, sol1.certificate) < 1e-8


def test_bound_inside_second_order_cones():
    """Bounds that cut SOCs: their norms are all-reduced across shards."""
    prob, d = fixture_prob("mixed")
    st = settings_from(d["settings"])
    # mixed: zero 4, nonneg 30, SOC 5, 5, 9 at rows 34..52, then PSD blocks
    m = prob[3].size
    bounds = np.array([0, 36, 47, m], np.int64)
    ws1, sol1, traj1 = single(prob, st)
    res, trajk = sharded(prob, st, 3, bounds=bounds)
    for k in sorted(traj1):
        assert rel(trajk[k], traj1[k]) < TOL, k
    assert all(s.status == sol1.status and s.info.iterations == sol1.info.iterations
               for _, s in res)


def test_big_soc_straddling_lasso():
    """LASSO with a 5002-dim SOC (chunked big-SOC path) split over 3 shards."""
    prob = G.gen_lasso(300, 5000, 60000, seed=3)
    st = P.Settings(max_iters=60)
    ws1, sol1, traj1 = single(prob, st, upto=60)
    res, trajk = sharded(prob, st, 3, upto=60)
    for k in sorted(traj1):
        assert rel(trajk[k], traj1[k]) < TOL, k
    assert all(s.status == sol1.status for _, s in res)


def test_nccl_one_rank_sharded_code_path():
    """The NCCL communicator itself (one rank) with every all-reduce point."""
    prob, d = fixture_prob("c1_lp_soc")
    st = settings_from(d["settings"], max_iters=200)
    ws1, sol1, traj1 = single(prob, st)
    lib = native.load()
    buf = (native.C.c_uint8 * 128)()
    native.check(lib.scs_nccl_unique_id(buf))
    colptr, rowidx, vals, b, c, cone = prob
    m = b.size
    spec = parallel.ShardSpec(0, 1, np.array([0, m], np.int64), nccl_id=bytes(buf), force=True)
    shard = parallel.shard_problem(colptr, rowidx, vals, b, c, cone, spec.bounds, 0)
    ws = P.Workspace(shard, st, dist=spec)
    traj = {}
    sol = ws.solve(on_iteration=lambda s: traj.__setitem__(s.iter, s.u.copy())
                   if s.iter <= 50 else None)
    for k in sorted(traj1):
        assert rel(traj[k], traj1[k]) < TOL, k
    assert sol.status == sol1.status and sol.info.iterations == sol1.info.iterations
    # the graph-launched loop (NCCL is capturable) gives the same answer
    sol2 = ws.solve()
    assert sol2.status == sol1.status and sol2.info.iterations == sol1.info.iterations


def test_shards_agree_on_the_streamed_format():
    """Production heuristic per shard (no SCS_STREAM knob): shard 0 holds
    5e6 nonzeros in dense tiles (it alone would stream), shard 1 3e6 (below
    the 4e6 gate).  The A^T pass's all-reduces follow its format (chunked when
    streamed), so both shards must choose the same -- here the CSR kernel --
    and the iterates equal the single-GPU solve's."""
    from paper_1312_3039_b200 import native
    rng = np.random.default_rng(17)
    m0, m1, n = 500_000, 500_000, 50_000
    rows = np.concatenate([rng.integers(0, m0, 5_200_000), m0 + rng.integers(0, m1, 3_000_000)])
    cols = rng.integers(0, n, rows.size)
    key = np.unique(cols.astype(np.int64) * (m0 + m1) + rows)
    cols, rows = np.divmod(key, m0 + m1)
    vals = rng.standard_normal(key.size)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    m = m0 + m1
    prob = (colptr, rows, vals, rng.standard_normal(m), rng.standard_normal(n), {"l": m})
    st = P.Settings(max_iters=8)
    ws1, sol1, traj1 = single(prob, st, upto=8)
    assert native.query(ws1._h, native.Q_FORMAT_A) == 1  # 8.2e6 nonzeros in one piece: streamed
    res, trajk = sharded(prob, st, 2, bounds=[0, m0, m], upto=8)
    fmts = {(native.query(ws._h, native.Q_FORMAT_A), native.query(ws._h, native.Q_FORMAT_AT))
            for ws, _ in res}
    assert fmts == {(0, 0)}, fmts
    for k in sorted(traj1):
        assert rel(trajk[k], traj1[k]) < TOL, (k, rel(trajk[k], traj1[k]))
