"""Pin the CPU oracle against the reference's own outputs (golden vectors).

CPU only.  Fixtures come from running conesplit 0.1.0 itself
(tests/golden/make_golden.py); the oracle must reproduce them before it is
trusted as the checker of the CUDA path.
"""

import math

import numpy as np
import pytest

from oracle import scs_oracle as O

from _fixtures import cones, eps_tuple, known_answers, load, names, rel

SLOW = {"c1_lp_soc", "c2_lp_infeasible", "mixed_nonorm_cgtol"}


def _solver(d, **over):
    st = dict(d["settings"])
    st.update(over)
    A = O.Csc(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"])
    return O.OracleSolver(A, d["b"], d["c"], d["cone"], alpha=st["alpha"],
                          max_iters=st["max_iters"], eps=eps_tuple(st),
                          check_interval=st["check_interval"], cg_max=st["cg_max"],
                          cg_tol=st["cg_tol"], normalize=st["normalize"],
                          sweeps=st["sweeps"])


@pytest.mark.parametrize("name", names())
def test_trajectory_and_solution(name):
    if name in SLOW:
        pytest.skip("slow case covered by test_slow_cases")
    _check(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(SLOW))
def test_slow_cases(name):
    _check(name)


def _check(name):
    d = load(name)
    s = _solver(d)
    # setup artefacts: equilibration and g = M^-1 h (scaling.py:79-129, embedding.py:145-162)
    assert rel(s.D, d["D"]) < 1e-13 and rel(s.E, d["E"]) < 1e-13
    assert math.isclose(s.sigma, float(d["sigma"]), rel_tol=1e-13)
    assert math.isclose(s.rho, float(d["rho"]), rel_tol=1e-13)
    assert rel(s.g, d["g"]) < 1e-12
    kept = list(d["kept"])
    got, norms, cgs, samp = {}, [], [], []
    sidx = d.get("sidx")

    def cb(k, u, v):
        if k in kept:
            got[k] = (u.copy(), v.copy())
        if k <= 50:
            norms.append((np.linalg.norm(u), np.linalg.norm(v)))
            cgs.append(s.cg_iters_total)
            if sidx is not None:
                samp.append((u[sidx].copy(), v[sidx].copy()))

    out = s.solve(on_iteration=cb)
    for i, k in enumerate(kept):
        assert rel(got[k][0], d["us"][i]) < 1e-12, (name, k)
        assert rel(got[k][1], d["vs"][i]) < 1e-12, (name, k)
    # every iterate k <= 50: norms, cumulative CG count, sampled entries
    np.testing.assert_allclose([a for a, _ in norms], d["unorm"], rtol=1e-12)
    np.testing.assert_allclose([b for _, b in norms], d["vnorm"], rtol=1e-12)
    np.testing.assert_array_equal(cgs, d["cg_total"])
    for k, (su, sv) in enumerate(samp):
        assert rel(su, d["us_sample"][k]) < 1e-12 and rel(sv, d["vs_sample"][k]) < 1e-12, k
    assert out["status"] == d["status"]
    assert out["iterations"] == d["iterations"]
    assert out["cg_iters"] == d["cg_iters"]
    # the reported Residuals of the last check (scaling.py:148-207)
    r = out["residuals"]
    fields = ("pri_norm", "dual_norm", "gap", "pri_thresh", "dual_thresh", "gap_thresh",
              "unbdd_measure", "infeas_measure")
    for i, (got_r, ref_r) in enumerate(zip([getattr(r, f) for f in fields], d["res"])):
        if np.isinf(ref_r):
            assert np.isinf(got_r), (name, i)
        else:  # the gap crosses zero: scaled by its threshold
            scale = max(abs(ref_r), abs(d["res"][5])) if i == 2 else abs(ref_r)
            assert abs(got_r - ref_r) <= 1e-9 * scale, (name, i)
    assert rel(out["u"], d["u_final"]) < 1e-9
    for key in ("x", "y", "s", "certificate"):
        if key in d:
            assert rel(out[key], d[key]) < 1e-9, key
    if d["status"] in ("solved", "max_iters_reached"):
        assert math.isclose(out["primal_obj"], float(d["primal_obj"]), rel_tol=1e-9)
        assert math.isclose(out["dual_obj"], float(d["dual_obj"]), rel_tol=1e-9)


def test_known_answers():
    ka = known_answers()
    A = O.Csc(2, 2, [0, 1, 2], [0, 1], [1.0, 2.0])
    assert O.mul(A, np.array([3.0, 4.0])).tolist() == ka["spmv"]
    E = O.Csc(2, 3, [0, 0, 0, 0], [], [])
    assert O.mul(E, np.ones(3)).tolist() == ka["spmv_empty"]
    A1 = O.Csc(1, 1, [0, 1], [0], [1.0])
    s = O.OracleSolver(A1, [1.0], [1.0], {"l": 1}, normalize=False)
    np.testing.assert_allclose(s.g, ka["setup_g"], atol=1e-12)
    assert math.isclose(s.denom, ka["setup_denom"], rel_tol=1e-12)
    s.cg_warm = np.zeros(1)
    np.testing.assert_allclose(s._kkt(np.array([1.0, 1.0]), 1e-9 * (1 + math.sqrt(2)), 110),
                               ka["solve_kkt"], atol=1e-12)
    s.cg_warm = np.zeros(1)
    w = np.array([1.0, 1.0, 1.0])
    rhs = w[:-1] - w[-1] * s.h
    p = s._kkt(rhs, 1e-9 * (1 + np.linalg.norm(rhs)), 110)
    uxy = p - (s.h @ p) / s.denom * s.g
    aff = np.concatenate([uxy, [w[-1] + s.c @ uxy[:1] + s.b @ uxy[1:]]])
    np.testing.assert_allclose(aff, ka["project_affine"], atol=1e-12)
    np.testing.assert_allclose(O.proj_soc(np.array([0.0, 3.0, 4.0])), ka["soc_boundary"], atol=1e-15)
    np.testing.assert_allclose(O.proj_soc(np.array([-5.0, 3.0, 4.0])), ka["soc_polar"])
    np.testing.assert_allclose(O.proj_embedding(np.array([-2.0, -1.0, -3.0]), 1, O.Cone(l=1)),
                               ka["embedding_basic"])
    np.testing.assert_allclose(O.proj_embedding(np.array([7.0, -1.0]), 0, O.Cone(z=1)),
                               ka["embedding_zero"])
    np.testing.assert_allclose(O.proj_primal_cone(np.array(ka["psd_diag_in"]), O.Cone(s=(2,))),
                               ka["psd_diag_out"], atol=1e-12)


def test_cone_projections_match_reference():
    data, specs = cones()
    for i, sp in enumerate(specs):
        cone = O.cone_from_spec(sp)
        for x, dref, pref in zip(data[f"x{i}"], data[f"dual{i}"], data[f"primal{i}"]):
            np.testing.assert_allclose(O.proj_dual_cone(x, cone), dref, rtol=0, atol=1e-11)
            np.testing.assert_allclose(O.proj_primal_cone(x, cone), pref, rtol=0, atol=1e-11)


def test_nonfinite_rejected():
    with pytest.raises(ValueError):
        O.proj_embedding(np.array([0.0, np.nan, 1.0]), 1, O.Cone(l=1))


def test_exp_cone_moreau_kkt():
    """Exp cone has no reference: check Moreau + KKT instead."""
    rng = np.random.default_rng(0)
    for _ in range(400):
        v = rng.standard_normal(3) * rng.choice([0.1, 1.0, 5.0])
        p = O.proj_exp_primal(v)
        d = p - v                      # -(polar part) must lie in K*
        scale = 1.0 + np.linalg.norm(v)
        assert abs(p @ d) <= 1e-9 * scale * scale
        r, s, t = p
        assert s >= -1e-12
        if s > 1e-10:
            assert s * math.exp(r / s) <= t + 1e-8 * scale
        u, vv, w = d
        if u < -1e-10:
            assert -u * math.exp(vv / u) <= math.e * w + 1e-8 * scale
        else:
            assert vv >= -1e-8 * scale and w >= -1e-8 * scale
        # Moreau: v = Pi_K(v) - Pi_K*(-v)
        np.testing.assert_allclose(p - O.proj_exp_dual(-v), v, atol=1e-9 * scale)
        # idempotence
        np.testing.assert_allclose(O.proj_exp_primal(p), p, atol=1e-9 * scale)


def test_oracle_pcg_reaches_reference_outcome():
    """Opt-in Jacobi PCG (not in the reference): same status and objectives
    within the solve tolerance as the reference's plain-CG solve."""
    d = load("ref_portfolio")
    s = _solver(d)
    s.precond = True
    s._rescale()
    s._refresh()
    out = s.solve()
    assert out["status"] == d["status"]
    tol = 10 * d["settings"]["eps_gap"]
    assert abs(out["primal_obj"] - float(d["primal_obj"])) <= tol * (1 + abs(float(d["primal_obj"])))
