"""Problem / solution files (problem_io.py): the
reference's JSON format read and re-written byte for byte (fixtures written
by conesplit's own fileio, tests/golden/make_io_golden.py), the same
FileFormatError members, and the binary .scsb layout round trip.  CPU only."""

import json
import os

import numpy as np
import pytest

import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import problem_io as io

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same_problem(a, b):
    assert (a.m, a.n) == (b.m, b.n)
    assert a.spec == b.spec
    for f in ("colptr", "rowidx", "vals"):
        np.testing.assert_array_equal(np.asarray(getattr(a.A, f)), np.asarray(getattr(b.A, f)))
    np.testing.assert_array_equal(a.b, b.b)
    np.testing.assert_array_equal(a.c, b.c)


def test_reference_json_problem_roundtrip_bytes(tmp_path):
    src = os.path.join(GOLD, "io_problem.json")
    data = io.read_problem(src)
    assert data.spec.psd_sides == (6,) and data.m == 49 and data.n == 39
    out = tmp_path / "p.json"
    io.write_problem(out, data)
    assert out.read_bytes() == open(src, "rb").read()


def test_reference_json_solution_roundtrip_bytes(tmp_path):
    src = os.path.join(GOLD, "io_solution.json")
    sol = io.read_solution(src)
    assert sol.status is P.Status.SOLVED and sol.x.size == 39
    out = tmp_path / "s.json"
    io.write_solution(out, sol)
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("mutate, member", [
    (lambda d: d.pop("m"), "m"),
    (lambda d: d.__setitem__("n", 1.5), "n"),
    (lambda d: d["A"].__setitem__("rowidx", [0.5]), "rowidx"),
    (lambda d: d["A"]["vals"].__setitem__(0, True), "vals"),
    (lambda d: d["A"]["rowidx"].__setitem__(0, 10**6), "A"),
    (lambda d: d["cone"].__setitem__("s", [-1]), "cone"),
    (lambda d: d.__setitem__("b", d["b"][:-1]), "b/c/cone"),
])
def test_json_errors_name_the_member(mutate, member):
    doc = json.load(open(os.path.join(GOLD, "io_problem.json")))
    mutate(doc)
    with pytest.raises(io.FileFormatError) as ei:
        io.problem_from_dict(doc)
    assert ei.value.member == member
    assert isinstance(ei.value, ValueError)


def test_bad_documents(tmp_path):
    p = tmp_path / "x.json"
    p.write_text("{not json")
    with pytest.raises(io.FileFormatError):
        io.read_problem(p)
    with pytest.raises(io.FileFormatError) as ei:
        io.solution_from_dict({"status": "great"})
    assert ei.value.member == "status"


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
    # the JSON form of the same problem agrees too (ep member when nonzero)
    j = tmp_path / "p.json"
    io.write_problem(j, data)
    _same_problem(io.read_problem(j), data)


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
