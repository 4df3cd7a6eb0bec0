"""GPU tests of the residual recurrence (SCS_RES_RECUR, default R = 32;
SCS_RES_RECUR_AT=0 keeps A^T u_y direct).

The termination check needs A u_x of the previous iterate (scaling.py:165).
Because v_x is exactly 0 after every iteration (the x-part cone is free),
u+_x = al (x - corr g_x) + (1 - al) u_x, so the solver carries
A u_x = al (A x - corr A g_x) + (1 - al) A u_x elementwise (k_cone_tail) and
computes it directly only every R iterations, in the merged first CG pass;
the other iterations run that pass on p alone (NV = 1).  The iterates never
read A u_x, so they must be bit-identical to the direct mode (R = 0); only
the residual values move, at rounding level.

A^T side (SCS_RES_RECUR_AT, default on): A^T A x is carried through the CG
Gp products (refreshed directly every R iterations), A^T rhs_y = F - A^T A x0
from the first pass's single product F, and A^T (v_y - u_y) follows
v+ - u+ = v - u_bar; A^T u_y = (A^T (u_y + v_y) - A^T (v_y - u_y)) / 2, so
the first A^T pass also runs with NV = 1.
"""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G

from _fixtures import load, rel

pytestmark = pytest.mark.gpu

NAMES = ["c1_lp_soc", "c2_lp_infeasible", "c2_lp_unbounded", "ref_portfolio", "mixed",
         "mixed_ci3_cg5"]


def fixture_data(d):
    st = d["settings"]
    settings = P.Settings(alpha=st["alpha"], max_iters=st["max_iters"], eps_pri=st["eps_pri"],
                          eps_dual=st["eps_dual"], eps_gap=st["eps_gap"],
                          eps_infeas=st["eps_infeas"], eps_unbdd=st["eps_unbdd"],
                          check_interval=st["check_interval"], cg_max=st["cg_max"],
                          cg_tol=st["cg_tol"], normalize=st["normalize"], sweeps=st["sweeps"])
    data = P.ProblemData(P.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"]),
                         d["b"], d["c"], P.ConeSpec.from_any(d["cone"]))
    return data, settings


def run(monkeypatch, data, settings, rec, env=()):
    monkeypatch.setenv("SCS_RES_RECUR", str(rec))
    for k, v in env:
        monkeypatch.setenv(k, v)
    traj = []
    sol = P.Workspace(data, settings).solve(
        on_iteration=lambda s: traj.append((s.u.copy(), s.v.copy())))
    return sol, traj


def _close(a, b, tol):
    if np.isnan(a) or np.isnan(b) or np.isinf(a) or np.isinf(b):  # no residual / no certificate
        return (np.isnan(a) and np.isnan(b)) or a == b
    return abs(a - b) <= tol * max(abs(a), abs(b), 1e-300)


@pytest.mark.parametrize("at", ["0", "1"])
@pytest.mark.parametrize("path", ["csr", "stream"])
@pytest.mark.parametrize("rec", [1, 3, 32])
@pytest.mark.parametrize("name", NAMES)
def test_recurrence_matches_direct(monkeypatch, name, rec, path, at):
    d = load(name)
    data, settings = fixture_data(d)
    env = [("SCS_STREAM", "1"), ("SCS_STREAM_W", "256")] if path == "stream" else []
    env.append(("SCS_RES_RECUR_AT", at))
    ref, tref = run(monkeypatch, data, settings, 0, env)
    got, tgot = run(monkeypatch, data, settings, rec, env)
    assert got.status == ref.status and got.info.iterations == ref.info.iterations
    assert len(tgot) == len(tref)
    # the iterates do not read A u_x: bit-identical on the CSR path with the
    # A side alone; on the streamed path the plain A p pass (NV = 1) runs on
    # another tile schedule than the merged NV = 2 pass (other split sums),
    # and with the A^T side the first pass's epilogue (and its ||r0||^2 sum)
    # runs in k_rows on another grid -- reduction-order changes: first 50
    # iterates to 1e-12
    for k, ((u0, v0), (u1, v1)) in enumerate(zip(tref, tgot)):
        if path == "csr" and at == "0":
            assert np.array_equal(u0, u1) and np.array_equal(v0, v1), k
        elif k < 50:
            assert rel(u1, u0) < 1e-12 and rel(v1, v0) < 1e-12, (k, rel(u1, u0))
    # residuals at the same final iterate (bit-identical runs): rounding level;
    # after a reduction-order change the final iterates themselves differ by
    # the trajectory's own drift (~1e-9 after thousands of iterations)
    tol = 1e-9 if (path == "csr" and at == "0") else 1e-6
    for key in ("pri_res", "dual_res", "gap"):
        assert _close(getattr(got.info, key), getattr(ref.info, key), tol), key
    for key in ("unbdd_measure", "infeas_measure"):
        assert _close(getattr(got.info.residuals, key), getattr(ref.info.residuals, key), tol), key
    assert got.status.value == d["status"]


def test_recurrence_lasso_long_run(monkeypatch):
    """Drift over many iterations stays at rounding level (|1 - alpha| < 1
    damps it; R = 1000 keeps the refresh out of the way)."""
    prob = G.gen_lasso(200, 4000, 40000, seed=5)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    st = P.Settings(max_iters=600, eps_pri=1e-9, eps_dual=1e-9, eps_gap=1e-9)
    ref, _ = run(monkeypatch, data, st, 0)
    got, _ = run(monkeypatch, data, st, 1000, [("SCS_RES_RECUR_AT", "0")])
    assert got.info.iterations == ref.info.iterations and got.status == ref.status
    assert np.array_equal(got.x, ref.x)
    for key in ("pri_res", "dual_res", "gap"):
        assert _close(getattr(got.info, key), getattr(ref.info, key), 1e-8), key
    # both sides: the A^T side's split epilogue changes the ||r0||^2 sum order
    got, _ = run(monkeypatch, data, st, 1000, [("SCS_RES_RECUR_AT", "1")])
    assert got.info.iterations == ref.info.iterations and got.status == ref.status
    assert rel(got.x, ref.x) < 1e-8
    for key in ("pri_res", "dual_res", "gap"):
        assert _close(getattr(got.info, key), getattr(ref.info, key), 1e-6), key


@pytest.mark.parametrize("world", [2, 3])
def test_recurrence_row_shards(monkeypatch, world):
    """Row shards: A u_x and A g_x are shard-local, no extra exchange."""
    from test_gpu_sharded import fixture_prob, settings_from, sharded
    prob, d = fixture_prob("c1_lp_soc")
    st = settings_from(d["settings"])
    monkeypatch.setenv("SCS_RES_RECUR", "0")
    res0, traj0 = sharded(prob, st, world)
    monkeypatch.setenv("SCS_RES_RECUR", "5")
    res1, traj1 = sharded(prob, st, world)
    for (_, s0), (_, s1) in zip(res0, res1):
        assert s0.status == s1.status and s0.info.iterations == s1.info.iterations
        assert s1.status.value == d["status"]
    for k in traj0:
        assert rel(traj1[k], traj0[k]) < 1e-12
