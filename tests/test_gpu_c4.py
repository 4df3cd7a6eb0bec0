"""Config 4 (BASELINE.json configs[3]): portfolio with SOC + exponential
cones + many small PSD blocks (generators.gen_portfolio_c4).

* small instance: trajectory vs the oracle to 1e-9 (exp/PSD parity is
  oracle-anchored), same status and iteration count;
* full size (1e5 assets, 11,111 PSD blocks, 1e4 exp cones): size-independent
  properties -- the solution passes the independent device checker, two
  runs are bitwise identical, and a 2-shard emulated run reproduces the
  single-GPU iterates to 1e-9.
"""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import check as CK
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import parallel
from oracle import scs_oracle as O

from _fixtures import rel

pytestmark = pytest.mark.gpu


def data_of(prob):
    colptr, rowidx, vals, b, c, cone = prob
    return P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))


def test_c4_small_vs_oracle():
    """First 50 iterates to 1e-9, then the state after 400 iterations."""
    prob = G.gen_portfolio_c4(60, 4, 10, seed=1)
    colptr, rowidx, vals, b, c, cone = prob
    A = O.Csc(b.size, colptr.size - 1, colptr, rowidx, vals)
    orc = O.OracleSolver(A, b, c, cone, max_iters=400, eps=(1e-5,) * 5)
    traj = {}
    ref = orc.solve(on_iteration=lambda k, u, v: traj.__setitem__(k, u.copy()) if k <= 50
                    else None)
    got = {}
    sol = P.Workspace(data_of(prob), P.Settings(max_iters=400, eps_pri=1e-5, eps_dual=1e-5,
                                                eps_gap=1e-5, eps_infeas=1e-5,
                                                eps_unbdd=1e-5)).solve(
        on_iteration=lambda s: got.__setitem__(s.iter, s.u.copy()))
    for k in sorted(traj):
        assert rel(got[k], traj[k]) < 1e-9, k
    assert sol.status.value == ref["status"]
    assert sol.info.iterations == ref["iterations"]
    assert rel(got[sol.info.iterations], ref["u"]) < 1e-8


@pytest.fixture(scope="module")
def c4_full():
    return G.gen_portfolio_c4(100_000, 10, 10_000, seed=1)


def test_c4_full_size_solves_and_checks(c4_full):
    data = data_of(c4_full)
    st = P.Settings(max_iters=20000)
    sol = P.Workspace(data, st).solve()
    assert sol.status is P.Status.SOLVED, sol.info
    ok, rows = CK.check_solution(data, sol, eps=5e-3)
    assert ok, [r for r in rows if not r[2]]


def test_c4_full_size_deterministic_and_shard_invariant(c4_full):
    data = data_of(c4_full)
    st = P.Settings(max_iters=20)
    runs = []
    for _ in range(2):
        traj = {}
        P.Workspace(data, st).solve(on_iteration=lambda s: traj.__setitem__(s.iter, s.u.copy()))
        runs.append(traj)
    assert all(np.array_equal(runs[0][k], runs[1][k]) for k in runs[0])
    n = c4_full[0].size - 1
    parts = {}
    parallel.emulated_solve(c4_full, st, 2, on_iteration=lambda r, s: parts.setdefault(
        s.iter, {}).__setitem__(r, s.u.copy()))
    for k, by in parts.items():
        u = np.concatenate([by[0][:n], by[0][n:-1], by[1][n:-1], by[0][-1:]])
        assert rel(u, runs[0][k]) < 1e-9, k
