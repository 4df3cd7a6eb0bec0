"""Binary problem files (problem_io.py): the .scsb layout
round trip, truncation and magic checks.  CPU only."""


import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import problem_io as io

def _same_problem(a, b):
    assert (a.m, a.n) == (b.m, b.n)
    assert a.spec == b.spec
    for f in ("colptr", "rowidx", "vals"):
        np.testing.assert_array_equal(np.asarray(getattr(a.A, f)), np.asarray(getattr(b.A, f)))
    np.testing.assert_array_equal(a.b, b.b)
    np.testing.assert_array_equal(a.c, b.c)


def test_json_not_handled(tmp_path):
    """The reference's JSON documents are out of scope."""
    colptr, rowidx, vals, b, c, cone = G.gen_lasso(10, 40, 300, seed=1)
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    with pytest.raises(ValueError):
        io.write_problem(tmp_path / "p.json", data)
    with pytest.raises(ValueError):
        io.read_problem(tmp_path / "p.json")


@pytest.mark.parametrize("maker", [
    lambda: G.gen_lasso(30, 100, 2000, seed=3),
    lambda: G.gen_cone_mix(n_psd=3, n_exp=4, n_soc=2, seed=1),
])
def test_binary_roundtrip(tmp_path, maker):
    colptr, rowidx, vals, b, c, cone = maker()
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    f = tmp_path / "p.scsb"
    io.write_problem(f, data)
    back = io.read_problem(f)
    _same_problem(back, data)


def test_binary_truncated_and_magic(tmp_path):
    colptr, rowidx, vals, b, c, cone = G.gen_lasso(10, 40, 300, seed=1)
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    f = tmp_path / "p.scsb"
    io.write_problem(f, data)
    raw = f.read_bytes()
    (tmp_path / "t.scsb").write_bytes(raw[:-16])
    with pytest.raises(io.FileFormatError):
        io.read_problem(tmp_path / "t.scsb")
    (tmp_path / "m.scsb").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(io.FileFormatError) as ei:
        io.read_problem(tmp_path / "m.scsb")
    assert ei.value.member == "<header>"
