"""GPU tests of the device checker (paper_1312_3039_b200/check.py,
csrc/check.cu) against the reference checker's own reports
(tests/golden/check_golden.npz) and, for exponential cones (no
reference), against the oracle restatement (oracle/check_oracle.py)."""

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import check as CK
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import native
from oracle import check_oracle as CO
from oracle import scs_oracle as O

from _fixtures import check_golden, load

pytestmark = pytest.mark.gpu

REPORTS = check_golden()


def data_of(d):
    return P.ProblemData(P.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"]),
                         d["b"], d["c"], P.ConeSpec.from_any(d["cone"]))


@pytest.mark.parametrize("rep", REPORTS, ids=[r["tag"] for r in REPORTS])
def test_device_checker_matches_reference_report(rep):
    d = load(rep["name"])
    data = data_of(d)
    sol = P.Solution(status=P.Status(rep["status"]), **rep["vecs"])
    ok, rows = CK.check_solution(data, sol, eps=rep["eps"])
    assert ok == rep["ok"]
    assert [r[0] for r in rows] == [r[0] for r in rep["rows"]]
    for (lab, v, good), (_, rv, rgood) in zip(rows, rep["rows"]):
        assert good == rgood, lab
        assert abs(v - rv) <= 1e-6 * abs(rv) + 1e-12, (lab, v, rv)


@pytest.mark.parametrize("dual", [False, True])
def test_margins_with_exp_and_psd_vs_oracle(dual):
    rng = np.random.default_rng(3)
    cone = {"z": 3, "l": 7, "q": [1, 4, 9], "s": [1, 3, 12, 40], "ep": 25}
    m = 3 + 7 + 14 + sum(k * (k + 1) // 2 for k in cone["s"]) + 75
    for _ in range(3):
        v = rng.standard_normal(m)
        got = native.cone_margins(v, cone, dual=dual)
        ref = [mg for _, mg in CO.membership_margins(v, cone, dual)]
        np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-11)


def test_margins_of_projected_points_are_nonnegative():
    cone = {"z": 0, "l": 5, "q": [6], "s": [5], "ep": 10}
    m = 5 + 6 + 15 + 30
    v = np.random.default_rng(1).standard_normal(m)
    p = native.project_cone(v, cone, kind="primal")
    mg = native.cone_margins(p, cone, dual=False)
    assert mg.min() >= -1e-12


def test_check_products_vs_oracle():
    prob = G.gen_lasso(200, 1000, 20000, seed=4)
    colptr, rowidx, vals, b, c, cone = prob
    A = P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals)
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(A.ncols), rng.standard_normal(A.nrows)
    ax, aty = native.check_products(A, x=x, y=y)
    Ao = O.Csc(b.size, colptr.size - 1, colptr, rowidx, vals)
    np.testing.assert_allclose(ax, O.mul(Ao, x), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(aty, O.mul_t(Ao, y), rtol=1e-12, atol=1e-12)


def test_check_our_own_c4_style_solution():
    """Solve a cone mix with exp cones and PSD blocks, then verify it."""
    prob = G.gen_cone_mix(n_psd=12, n_exp=10, n_soc=4, soc_dim=5, l=40, z=3, n=50,
                          nnz_per_col=6, seed=0)
    colptr, rowidx, vals, b, c, cone = prob
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    sol = P.solve(data, P.Settings(max_iters=2000, eps_pri=1e-6, eps_dual=1e-6, eps_gap=1e-6))
    assert sol.status is P.Status.SOLVED
    ok, rows = CK.check_solution(data, sol, eps=1e-4)
    assert ok, [r for r in rows if not r[2]]
    A = O.Csc(b.size, colptr.size - 1, colptr, rowidx, vals)
    ok2, rows2 = CO.check(A, b, c, cone, "solved", 1e-4, x=sol.x, y=sol.y, s=sol.s)
    assert ok2 == ok
    for (lab, v, _), (_, rv, _) in zip(rows, rows2):
        assert abs(v - rv) <= 1e-9 * (1 + abs(rv)), lab
