"""GPU parity: the CUDA path through the C-ABI against the reference's golden
fixtures (produced by conesplit itself) and against the CPU oracle on the
same seeded inputs.

Bars (BASELINE.json north star): identical status; objectives within 1e-6
relative; x, y, s within 1e-5 relative at eps=1e-5; the first 50 (u, v)
iterates within 1e-9 relative.  Exp-cone cases have no reference (SURVEY
D2) and are checked against the oracle and through KKT / Moreau properties.
"""

import math

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import native
from oracle import scs_oracle as O

from _fixtures import cones as cone_fixture
from _fixtures import eps_tuple, known_answers, load, names, rel

pytestmark = pytest.mark.gpu

ITERATE_TOL = 1e-9
OBJ_TOL = 1e-6
VEC_TOL = 1e-5


def settings_from(st, **over):
    kw = dict(alpha=st["alpha"], max_iters=st["max_iters"], eps_pri=st["eps_pri"],
              eps_dual=st["eps_dual"], eps_gap=st["eps_gap"], eps_infeas=st["eps_infeas"],
              eps_unbdd=st["eps_unbdd"], check_interval=st["check_interval"],
              cg_max=st["cg_max"], cg_tol=st["cg_tol"], normalize=st["normalize"],
              sweeps=st["sweeps"], linsys_mode="indirect")
    kw.update(over)
    return P.Settings(**kw)


def problem(colptr, rowidx, vals, b, c, cone):
    m, n = b.size, colptr.size - 1
    return P.ProblemData(P.SparseMatrix(m, n, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))


def fixture_problem(d):
    return problem(d["colptr"], d["rowidx"], d["vals"], d["b"], d["c"], d["cone"])


def _vec_close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) <= tol * max(np.linalg.norm(b), 1.0)


# Unnormalised problem with a fixed absolute cg_tol: the reference itself is
# chaotic here -- injecting 1-ulp noise into its SpMV outputs moves its own
# iterates by 1.4e-9 at iteration 30 and 1.6e-7 at iteration 50 (see
# DESIGN.md, parity).  Trajectory checked to iteration 20; after that only
# the iteration count and a post-loop status (solver.py:364-369) -- which
# the reference itself does not reproduce under 1-ulp noise -- are checked.
TRAJ_ONLY = {"mixed_nonorm_cgtol": 20}
# Residual tolerance: the default residual recurrences carry
# A u_x and A^T u_y at rounding level between direct refreshes.
RES_TOL = 1e-7


def _res_close(got, ref, tol, what):
    for i, (g, r) in enumerate(zip(got, ref)):
        if math.isinf(r):
            assert math.isinf(g), (what, i, g, r)
            continue
        scale = max(abs(r), abs(ref[5])) if i == 2 else abs(r)  # the gap crosses zero
        assert abs(g - r) <= tol * max(scale, 1e-300), (what, i, g, r)


@pytest.mark.parametrize("name", names())
def test_golden_solve(name):
    d = load(name)
    st = settings_from(d["settings"])
    ws = P.Workspace(fixture_problem(d), st)
    sc = ws.scal
    assert rel(sc.D, d["D"]) < 1e-12 and rel(sc.E, d["E"]) < 1e-12
    assert math.isclose(sc.sigma, float(d["sigma"]), rel_tol=1e-12)
    assert math.isclose(sc.rho, float(d["rho"]), rel_tol=1e-12)
    kept = [int(k) for k in d["kept"]]
    sidx = d.get("sidx")
    got, norms, cgs, samp = {}, [], [], []

    def cb(state):
        k = state.iter
        if k in kept:
            got[k] = (state.u.copy(), state.v.copy())
        if k <= 50:
            norms.append((np.linalg.norm(state.u), np.linalg.norm(state.v)))
            cgs.append(ws.cache.cg_iters_total)
            if sidx is not None:
                samp.append((state.u[sidx].copy(), state.v[sidx].copy()))

    sol = ws.solve(on_iteration=cb)
    lim = TRAJ_ONLY.get(name, 10**9)
    # every iterate k <= 50 (north star: first 50 iterates within 1e-9)
    for i, k in enumerate(kept):
        if k > lim:
            continue
        assert rel(got[k][0], d["us"][i]) < ITERATE_TOL, (name, k, rel(got[k][0], d["us"][i]))
        assert rel(got[k][1], d["vs"][i]) < ITERATE_TOL, (name, k)
    for k in range(min(len(norms), lim)):
        assert abs(norms[k][0] - d["unorm"][k]) <= ITERATE_TOL * d["unorm"][k], (name, k)
        assert abs(norms[k][1] - d["vnorm"][k]) <= ITERATE_TOL * d["vnorm"][k], (name, k)
    for k in range(min(len(samp), lim)):
        assert rel(samp[k][0], d["us_sample"][k]) < ITERATE_TOL, (name, k)
        assert rel(samp[k][1], d["vs_sample"][k]) < ITERATE_TOL, (name, k)
    if name in TRAJ_ONLY:
        # the reference's own post-loop status flips under 1-ulp SpMV noise
        # here (3 of 6 noisy runs end max_iters_reached instead of
        # indeterminate: tools/ref_noise_status.py); the rule itself is
        # pinned by the maxit_* / indet_* fixtures
        assert sol.status.value in ("indeterminate", "max_iters_reached")
        assert sol.info.iterations == d["iterations"]
        return
    # status: exact, including the post-loop MAX_ITERS_REACHED / INDETERMINATE rule
    assert sol.status.value == d["status"], (name, sol.status, d["status"])
    assert len(norms) == min(50, d["iterations"])
    # cumulative CG count (setup solve of g included, embedding.py:112) after
    # every iteration, and the reported total (solver.py:376)
    np.testing.assert_array_equal(cgs, d["cg_total"])
    assert sol.info.cg_iters == d["cg_iters"], (sol.info.cg_iters, d["cg_iters"])
    # iteration count: exact
    assert sol.info.iterations == d["iterations"], (sol.info.iterations, d["iterations"])
    # the reported Residuals of the final check (scaling.py:148-207, solver.py:375)
    _res_close([getattr(sol.info.residuals, f) for f in RES_FIELDS], d["res"], RES_TOL, name)
    if d["status"] in ("solved", "max_iters_reached"):
        for key, ref in (("primal_obj", d["primal_obj"]), ("dual_obj", d["dual_obj"])):
            assert abs(getattr(sol, key) - float(ref)) <= OBJ_TOL * max(1.0, abs(float(ref))), key
        for key in ("x", "y", "s"):
            assert _vec_close(getattr(sol, key), d[key], VEC_TOL), key
    elif d["status"] != "indeterminate":
        assert _vec_close(sol.certificate, d["certificate"], VEC_TOL)


RES_FIELDS = ("pri_norm", "dual_norm", "gap", "pri_thresh", "dual_thresh", "gap_thresh",
              "unbdd_measure", "infeas_measure")  # scaling.py:48-55


@pytest.mark.parametrize("name", ["c1_lp_soc", "c2_lp_infeasible", "c2_lp_unbounded",
                                  "ref_portfolio", "mixed"])
def test_golden_fast_path_matches(name):
    """The graph-launched solve (no per-iteration host callback) must give
    the same answer as the stepping path above."""
    d = load(name)
    sol = P.solve(fixture_problem(d), settings_from(d["settings"]))
    assert sol.status.value == d["status"]
    assert sol.info.iterations == d["iterations"]
    assert sol.info.cg_iters == d["cg_iters"]
    if d["status"] == "solved":
        assert abs(sol.objective - 0.5 * (float(d["primal_obj"]) + float(d["dual_obj"]))) <= \
            OBJ_TOL * max(1.0, abs(float(d["primal_obj"])))
    d2 = P.solution_to_dict(sol)
    assert d2["status"] == d["status"] and d2["info"]["iters"] == sol.info.iterations


def test_known_answers_device():
    ka = known_answers()
    A = P.SparseMatrix.from_dense([[1.0, 0.0], [0.0, 2.0]])
    data = P.ProblemData(A, np.array([1.0, 1.0]), np.array([1.0, 1.0]), P.ConeSpec(nonneg_dim=2))
    ws = P.Workspace(data, P.Settings(normalize=False))
    np.testing.assert_array_equal(ws.apply_a([3.0, 4.0]), ka["spmv"])
    np.testing.assert_array_equal(ws.apply_a([1.0, 2.0], transpose=True), [1.0, 4.0])
    e = P.ProblemData(P.SparseMatrix(2, 3, np.zeros(4, np.int64), [], []), np.zeros(2),
                      np.zeros(3), P.ConeSpec(nonneg_dim=2))
    we = P.Workspace(e, P.Settings(normalize=False))
    np.testing.assert_array_equal(we.apply_a(np.ones(3)), ka["spmv_empty"])


def test_cone_projection_fixture():
    data, specs = cone_fixture()
    for i, sp in enumerate(specs):
        cone = dict(sp, ep=0)
        for x, dref, pref in zip(data[f"x{i}"], data[f"dual{i}"], data[f"primal{i}"]):
            np.testing.assert_allclose(native.project_cone(x, cone, "dual"), dref, atol=1e-11)
            np.testing.assert_allclose(native.project_cone(x, cone, "primal"), pref, atol=1e-10)


def test_cone_known_answers():
    ka = known_answers()
    np.testing.assert_allclose(native.project_cone([0.0, 3.0, 4.0], {"q": [3]}, "primal"),
                               ka["soc_boundary"], atol=1e-14)
    np.testing.assert_allclose(native.project_cone([-5.0, 3.0, 4.0], {"q": [3]}, "primal"),
                               ka["soc_polar"], atol=1e-14)
    np.testing.assert_allclose(native.project_cone([-2.0, -1.0, -3.0], {"l": 1}, "embedding", n=1),
                               ka["embedding_basic"])
    np.testing.assert_allclose(native.project_cone([7.0, -1.0], {"z": 1}, "embedding", n=0),
                               ka["embedding_zero"])
    np.testing.assert_allclose(native.project_cone(ka["psd_diag_in"], {"s": [2]}, "primal"),
                               ka["psd_diag_out"], atol=1e-12)
    with pytest.raises(native.NativeError):
        native.project_cone([np.nan, 1.0], {"l": 2}, "dual")


def test_big_soc_and_psd_sides_vs_oracle():
    rng = np.random.default_rng(3)
    cone = {"z": 5, "l": 100, "q": [3000, 20000, 2049, 2048, 1], "s": [1, 2, 7, 16, 33, 64, 100],
            "ep": 7}
    oc = O.cone_from_spec(cone)
    for scale in (0.5, 3.0):
        x = scale * rng.standard_normal(oc.dim)
        got = native.project_cone(x, cone, "dual")
        exp = O.proj_dual_cone(x, oc)
        np.testing.assert_allclose(got, exp, atol=1e-9 * (1 + np.abs(x).max()))


def test_exp_cone_device_kkt():
    rng = np.random.default_rng(11)
    V = rng.standard_normal((2000, 3)) * rng.choice([0.05, 1.0, 20.0], size=(2000, 1))
    out = native.project_cone(V.ravel(), {"ep": 2000}, "primal").reshape(-1, 3)
    for v, p in zip(V, out):
        ref = O.proj_exp_primal(v)
        scale = 1.0 + np.linalg.norm(v)
        assert np.linalg.norm(p - ref) <= 1e-8 * scale, (v, p, ref)


@pytest.mark.parametrize("seed", [0, 1])
def test_cone_mix_with_exp_vs_oracle(seed):
    """C4-style mix (zero, nonneg, SOC, many small PSD, exp): no reference for
    exp cones, so the oracle is the checker; trajectories to 1e-9."""
    prob = G.gen_cone_mix(n_psd=12, n_exp=10, n_soc=4, soc_dim=5, l=40, z=3, n=50,
                          nnz_per_col=6, seed=seed)
    colptr, rowidx, vals, b, c, cone = prob
    st = P.Settings(max_iters=400, eps_pri=1e-5, eps_dual=1e-5, eps_gap=1e-5)
    A = O.Csc(b.size, colptr.size - 1, colptr, rowidx, vals)
    orc = O.OracleSolver(A, b, c, cone, max_iters=400, eps=(1e-5,) * 5)
    traj = {}
    ref = orc.solve(on_iteration=lambda k, u, v: traj.__setitem__(k, (u.copy(), v.copy()))
                    if k <= 50 else None)
    got = {}
    ws = P.Workspace(problem(*prob), st)
    sol = ws.solve(on_iteration=lambda s: got.__setitem__(s.iter, (s.u.copy(), s.v.copy()))
                   if s.iter <= 50 else None)
    for k in sorted(set(traj) & set(got)):
        assert rel(got[k][0], traj[k][0]) < ITERATE_TOL, k
    assert sol.status.value == ref["status"]
    assert abs(sol.info.iterations - ref["iterations"]) <= 2


def test_lasso_vs_oracle_trajectory():
    prob = G.gen_lasso(200, 1000, 20000, seed=4)
    colptr, rowidx, vals, b, c, cone = prob
    A = O.Csc(b.size, colptr.size - 1, colptr, rowidx, vals)
    orc = O.OracleSolver(A, b, c, cone, max_iters=50)
    traj = {}
    orc.solve(on_iteration=lambda k, u, v: traj.__setitem__(k, u.copy()))
    got = {}
    ws = P.Workspace(problem(*prob), P.Settings(max_iters=50))
    ws.solve(on_iteration=lambda s: got.__setitem__(s.iter, s.u.copy()))
    for k in traj:
        assert rel(got[k], traj[k]) < ITERATE_TOL, k


def test_warm_start_and_update_vectors():
    d = load("ref_lp_feasible")
    prob = fixture_problem(d)
    st = P.Settings()
    ws = P.Workspace(prob, st)
    sol = ws.solve()
    assert sol.status is P.Status.SOLVED
    # warm start at its own solution (solver.py:345-348); the reference
    # needs 117 iterations here (not SPEC criterion 12's 25), and so must we
    sol2 = ws.solve(warm_start=(sol.x, sol.y, sol.s))
    A = O.Csc(prob.m, prob.n, prob.A.colptr, prob.A.rowidx, prob.A.vals)
    orc = O.OracleSolver(A, prob.b, prob.c, {"l": prob.m})
    ref2 = orc.solve(warm_start=(sol.x, sol.y, sol.s))
    assert sol2.status is P.Status.SOLVED
    assert abs(ref2["iterations"] - sol2.info.iterations) <= 1
    assert sol2.info.iterations < sol.info.iterations
    # update_vectors keeps A; equals a fresh workspace on the new data
    b2 = prob.b * 1.1
    ws.update_vectors(b=b2)
    s3 = ws.solve()
    s4 = P.solve(P.ProblemData(prob.A, b2, prob.c, prob.spec), st)
    assert s3.status == s4.status and s3.info.iterations == s4.info.iterations
    assert abs(s3.objective - s4.objective) <= 1e-9 * max(1, abs(s4.objective))


def test_error_behaviour():
    with pytest.raises(ValueError):
        P.Settings(alpha=2.0)
    with pytest.raises(ValueError):
        P.Settings(linsys_mode="direct")
    A = P.SparseMatrix.from_dense([[1.0]])
    with pytest.raises(ValueError):
        P.ProblemData(A, np.array([np.inf]), np.array([1.0]), P.ConeSpec(nonneg_dim=1))
    with pytest.raises(ValueError):
        P.ProblemData(A, np.array([1.0]), np.array([1.0]), P.ConeSpec(nonneg_dim=2))


def test_north_star_signature_and_dict():
    d = load("tiny_lp")
    A = P.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"])
    sol = P.solve(A, d["b"], d["c"], {"z": 0, "l": 1, "q": [], "s": []},
                  P.Settings(linsys_mode="indirect"))
    assert sol.status.value == d["status"] and sol.info.iterations == d["iterations"]
    doc = P.solution_to_dict(sol)
    assert set(doc) >= {"status", "x", "y", "s", "info"}
    assert abs(doc["x"][0] - float(d["x"][0])) < 1e-9


@pytest.mark.parametrize("sides", [[300], [600, 2, 257]])
def test_large_psd_sides_vs_eigh(sides):
    """PSD blocks beyond the shared-memory side (and beyond 128 rotation
    pairs): matrices and pair arrays in global scratch.  The projection is
    unique, so numpy's eigh (not the pure-Python Jacobi restatement, too
    slow at these sides) is the checker."""
    rng = np.random.default_rng(sum(sides))
    cone = {"s": sides}
    oc = O.cone_from_spec(cone)
    x = rng.standard_normal(oc.dim)
    got = native.project_cone(x, cone, "dual")
    off = 0
    for k in sides:
        d = k * (k + 1) // 2
        m = O.svec_to_mat(x[off:off + d], k)
        w, v = np.linalg.eigh(0.5 * (m + m.T))
        exp = O.mat_to_svec((v * np.maximum(w, 0.0)) @ v.T)
        np.testing.assert_allclose(got[off:off + d], exp, atol=1e-9 * (1 + np.abs(x).max()))
        off += d


@pytest.mark.parametrize("name", ["c1_lp_soc", "c2_lp_unbounded", "maxit_lasso_q18p",
                                  "ref_portfolio"])
def test_device_loop_matches_host_loop(name, monkeypatch):
    """One solve = one launch of the device-side loop graph (WHILE node over
    a SWITCH of the refresh / non-refresh iteration graphs) must give the
    same bits as the host-driven loop over the same iteration graphs
    (SCS_LOOP_GRAPH=0), and stop on the same iteration."""
    d = load(name)
    st = settings_from(d["settings"])
    sols = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SCS_LOOP_GRAPH", flag)
        ws = P.Workspace(fixture_problem(d), st)
        sols.append((ws.solve(), ws.final_state))
    (a, fa), (b, fb) = sols
    assert a.status == b.status and a.info.iterations == b.info.iterations == d["iterations"]
    assert a.info.cg_iters == b.info.cg_iters == d["cg_iters"]
    assert np.array_equal(fa.u, fb.u) and np.array_equal(fa.v, fb.v)
    for key in ("x", "y", "s", "certificate"):
        va, vb = getattr(a, key), getattr(b, key)
        assert (va is None) == (vb is None)
        if va is not None:
            assert np.array_equal(va, vb), key


def test_pinned_buffers_roundtrip():
    """Warm start from page-locked host buffers, solution returned in pooled
    page-locked buffers (recycled after the arrays die)."""
    d = load("ref_lp_feasible")
    ws = P.Workspace(fixture_problem(d), settings_from(d["settings"]))
    sol = ws.solve()
    x0, y0, s0 = P.pinned_empty(d["n"]), P.pinned_empty(d["m"]), P.pinned_empty(d["m"])
    x0[:], y0[:], s0[:] = sol.x, sol.y, sol.s
    again = ws.solve(warm_start=(x0, y0, s0))
    plain = ws.solve(warm_start=(np.array(sol.x), np.array(sol.y), np.array(sol.s)))
    assert again.info.iterations == plain.info.iterations
    assert np.array_equal(again.x, plain.x) and np.array_equal(again.y, plain.y)


def test_query_and_cache_counter():
    """scs_query: the production format switch (CSR below 4e6 nonzeros), the
    per-iteration launch count, and EmbeddingCache.cg_iters_total kept in
    step with the reference's (setup solve, then every solve; update_vectors
    re-solves g, embedding.py:145-162)."""
    d = load("ref_lp_feasible")
    ws = P.Workspace(fixture_problem(d), settings_from(d["settings"]))
    h = ws._h
    assert native.query(h, native.Q_FORMAT_A) == 0 and native.query(h, native.Q_FORMAT_AT) == 0
    assert native.query(h, native.Q_STREAM_BYTES_A) == 0
    assert native.query(h, native.Q_LAUNCHES_PER_ITER) > 0
    setup_cg = ws.cache.cg_iters_total
    assert setup_cg > 0
    sol = ws.solve()
    assert ws.cache.cg_iters_total == sol.info.cg_iters == d["cg_iters"]
    ws.update_vectors(b=d["b"])
    assert ws.cache.cg_iters_total > sol.info.cg_iters
    with pytest.raises(native.NativeError):
        native.query(h, 99)


def test_pinned_pool_recycles():
    """Pooled page-locked buffers return to the pool when their arrays die."""
    import gc
    a = P.pinned_empty(1000)
    addr = a.ctypes.data
    del a
    gc.collect()
    b = P.pinned_zeros(1000)
    assert b.ctypes.data == addr and not b.any()


@pytest.mark.parametrize("split", ["0", "1"])
def test_split_long_rows_vs_oracle(monkeypatch, split):
    """Rows split into pieces (SCS_SPLIT=1: every row longer than the piece
    cap; the portfolio's budget row of 3000 assets has > 32 pieces and is
    summed by one warp inside k_rows) against the oracle's iterates, and the
    unsplit CSR path (SCS_SPLIT=0) against the same."""
    monkeypatch.setenv("SCS_SPLIT", split)
    colptr, rowidx, vals, b, c, cone = G.gen_portfolio_c4(3000, 5, 0, n_groups=0, seed=3)
    cone = {k: v for k, v in cone.items() if k != "ep"}
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    A = O.Csc(b.size, colptr.size - 1, colptr, rowidx, vals)
    orc = O.OracleSolver(A, b, c, cone, max_iters=30)
    ref = {}
    orc.solve(on_iteration=lambda k, u, v: ref.__setitem__(k, u.copy()))
    got = {}
    P.Workspace(data, P.Settings(max_iters=30)).solve(
        on_iteration=lambda s: got.__setitem__(s.iter, s.u.copy()))
    assert sorted(got) == sorted(ref)
    for k in ref:
        assert rel(got[k], ref[k]) < 1e-9, (split, k, rel(got[k], ref[k]))
