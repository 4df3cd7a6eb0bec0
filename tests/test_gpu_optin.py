"""GPU tests of the opt-in modes (include/scs_b200.h
SCS_FAST_*), which are reported separately from parity mode.

* precond (Jacobi PCG, the north star's "diagonally preconditioned CG"):
  not in the reference, so parity is against the oracle's PCG restatement
  (trajectories to 1e-9, same status and iteration count) and, for the
  outcome, against the reference's own fixtures (same status, objectives
  to 1e-6 -- SURVEY D1 measured exactly this for a Jacobi PCG).
* fast (A x by recurrence): a rounding-level change, so the reference's
  own first-50 iterates must still agree to 1e-9.
"""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from oracle import scs_oracle as O

from _fixtures import eps_tuple, load, rel

pytestmark = pytest.mark.gpu

CASES = ["c1_lp_soc", "mixed", "ref_portfolio", "ref_lasso", "ref_lp_infeasible",
         "ref_lp_unbounded"]


def settings_from(st, **over):
    kw = dict(alpha=st["alpha"], max_iters=st["max_iters"], eps_pri=st["eps_pri"],
              eps_dual=st["eps_dual"], eps_gap=st["eps_gap"], eps_infeas=st["eps_infeas"],
              eps_unbdd=st["eps_unbdd"], check_interval=st["check_interval"],
              cg_max=st["cg_max"], cg_tol=st["cg_tol"], normalize=st["normalize"],
              sweeps=st["sweeps"])
    kw.update(over)
    return P.Settings(**kw)


def data_of(d):
    return P.ProblemData(P.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"]),
                         d["b"], d["c"], P.ConeSpec.from_any(d["cone"]))


def run(data, st, upto=50):
    got = {}
    sol = P.Workspace(data, st).solve(
        on_iteration=lambda s: got.__setitem__(s.iter, s.u.copy()) if s.iter <= upto else None)
    return sol, got


@pytest.mark.parametrize("name", CASES)
def test_pcg_matches_oracle_pcg(name):
    d = load(name)
    st = d["settings"]
    A = O.Csc(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"])
    orc = O.OracleSolver(A, d["b"], d["c"], d["cone"], alpha=st["alpha"],
                         max_iters=st["max_iters"], eps=eps_tuple(st),
                         check_interval=st["check_interval"], cg_max=st["cg_max"],
                         cg_tol=st["cg_tol"], normalize=st["normalize"], sweeps=st["sweeps"],
                         precond=True)
    traj = {}
    ref = orc.solve(on_iteration=lambda k, u, v: traj.__setitem__(k, u.copy()) if k <= 50
                    else None)
    sol, got = run(data_of(d), settings_from(st, precond=True))
    for k in sorted(traj):
        assert rel(got[k], traj[k]) < 1e-9, (name, k, rel(got[k], traj[k]))
    assert sol.status.value == ref["status"]
    assert abs(sol.info.iterations - ref["iterations"]) <= max(2, ref["iterations"] // 200)
    # the outcome agrees with the reference's (unpreconditioned) solve
    assert sol.status.value == d["status"]
    if d["status"] == "solved":
        tol = 10 * d["settings"]["eps_gap"]
        for key in ("primal_obj", "dual_obj"):
            assert abs(getattr(sol, key) - float(d[key])) <= tol * (1.0 + abs(float(d[key]))), key


@pytest.mark.parametrize("name", CASES + ["c2_lp_unbounded"])
def test_recurrence_keeps_reference_iterates(name):
    d = load(name)
    sol, got = run(data_of(d), settings_from(d["settings"], fast=True))
    kept = [int(k) for k in d["kept"]]
    for i, k in enumerate(kept):
        assert rel(got[k], d["us"][i]) < 1e-9, (name, k, rel(got[k], d["us"][i]))
    assert sol.status.value == d["status"]
    assert abs(sol.info.iterations - d["iterations"]) <= max(2, d["iterations"] // 200)


def test_recurrence_refresh_bounds_drift(monkeypatch):
    """Long LASSO run: recurrence (refresh every 20, and never) vs direct."""
    prob = G.gen_lasso(200, 1000, 20000, seed=4)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    st = dict(max_iters=300, eps_pri=1e-7, eps_dual=1e-7, eps_gap=1e-7)
    base, tb = run(data, P.Settings(**st), upto=300)
    fast, tf = run(data, P.Settings(fast=True, **st), upto=300)
    worst = max(rel(tf[k], tb[k]) for k in tb)
    assert worst < 1e-9, worst
    assert fast.status == base.status and fast.info.iterations == base.info.iterations
    monkeypatch.setenv("SCS_RECUR_REFRESH", "100000")  # never refresh: drift stays small
    never, tn = run(data, P.Settings(fast=True, **st), upto=300)
    assert max(rel(tn[k], tb[k]) for k in tb) < 1e-7


def test_pcg_and_recurrence_together():
    d = load("c1_lp_soc")
    sol, _ = run(data_of(d), settings_from(d["settings"], precond=True, fast=True))
    assert sol.status.value == d["status"]
    assert abs(sol.primal_obj - float(d["primal_obj"])) <= 1e-5 * max(1, abs(float(d["primal_obj"])))
