"""Pin the CPU restatement of the reference checker (oracle/check_oracle.py)
against the reference's own reports (tests/golden/check_golden.npz)."""

import numpy as np
import pytest

from oracle import check_oracle as CO
from oracle import scs_oracle as O

from _fixtures import check_golden, load

REPORTS = check_golden()


@pytest.mark.parametrize("rep", REPORTS, ids=[r["tag"] for r in REPORTS])
def test_oracle_checker_matches_reference_report(rep):
    d = load(rep["name"])
    A = O.Csc(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"])
    ok, rows = CO.check(A, d["b"], d["c"], d["cone"], rep["status"], rep["eps"], **rep["vecs"])
    assert ok == rep["ok"]
    assert [r[0] for r in rows] == [r[0] for r in rep["rows"]]
    for (lab, v, good), (_, rv, rgood) in zip(rows, rep["rows"]):
        assert good == rgood, lab
        # the reference prints 7 significant digits
        assert abs(v - rv) <= 1e-6 * abs(rv) + 1e-12, (lab, v, rv)


def test_reports_cover_violations():
    assert any(not r["ok"] for r in REPORTS) and any(r["ok"] for r in REPORTS)
    kinds = {r["status"] for r in REPORTS}
    assert {"solved", "infeasible", "unbounded"} <= kinds
