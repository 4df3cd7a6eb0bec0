"""CPU checks of the native boundary: the library loads, exports every
symbol include/scs_b200.h declares, and its host-only entry points (the
LASSO generator and the row partitioner) behave.  No CUDA calls."""

import os
import re

import numpy as np
import pytest

from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "scs_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(scs_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = native.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(native.EXPORTS)
    assert lib.scs_abi_version() == 2


def test_last_error_without_handle():
    lib = native.load()
    assert isinstance(lib.scs_last_error(None), bytes)


@pytest.mark.parametrize("threads", [1, 3])
def test_gen_lasso_encoding(threads):
    p, q, nnzf = 12, 40, 100
    colptr, rowidx, vals, b, c, cone = native.gen_lasso(p, q, nnzf, seed=5, threads=threads)
    m, n = 2 * p + q + 2, 2 * p + 1
    assert colptr.size == n + 1 and b.size == m and c.size == n
    assert rowidx.size == 4 * p + 2 + nnzf
    # CSC invariants (sparse_linalg.py:34-54)
    for j in range(n):
        r = rowidx[colptr[j]:colptr[j + 1]]
        assert np.all(np.diff(r) > 0) and (r.size == 0 or (r[0] >= 0 and r[-1] < m))
    A = np.zeros((m, n))
    cols = np.repeat(np.arange(n), np.diff(colptr))
    A[rowidx, cols] = vals
    idx = np.arange(p)
    # -t <= z <= t rows and the SOC head (generators.py:87-110)
    assert np.all(A[idx, idx] == 1) and np.all(A[idx, p + idx] == -1)
    assert np.all(A[p + idx, idx] == -1) and np.all(A[p + idx, p + idx] == -1)
    assert A[2 * p, 2 * p] == -1 and A[2 * p + 1, 2 * p] == 1
    assert b[2 * p] == 1 and b[2 * p + 1] == 1
    F = A[2 * p + 2:, :p] / 2.0
    assert np.count_nonzero(F) == nnzf
    # mu = 0.1 ||F^T g||_inf with g = b_F / 2 (generators.py:78-79)
    g = b[2 * p + 2:] / 2.0
    assert np.isclose(c[p], 0.1 * np.max(np.abs(F.T @ g)))
    assert np.all(c[:p] == 0) and c[-1] == 0.5
    assert cone == {"z": 0, "l": 2 * p, "q": [q + 2], "s": [], "ep": 0}


def test_gen_lasso_thread_independent_and_sliced():
    full = native.gen_lasso(20, 50, 300, seed=9, threads=1)
    again = native.gen_lasso(20, 50, 300, seed=9, threads=4)
    for a, b in zip(full[:5], again[:5]):
        np.testing.assert_array_equal(a, b)
    m = 2 * 20 + 50 + 2
    colptr, rowidx, vals, b, c, _ = full
    cols = np.repeat(np.arange(colptr.size - 1), np.diff(colptr))
    for lo, hi in ((0, 37), (37, 60), (60, m)):
        cp, ri, va, bb, cc, _ = native.gen_lasso(20, 50, 300, seed=9, row_lo=lo, row_hi=hi)
        keep = (rowidx >= lo) & (rowidx < hi)
        cs = np.repeat(np.arange(cp.size - 1), np.diff(cp))
        np.testing.assert_array_equal(cs, cols[keep])
        np.testing.assert_array_equal(ri, rowidx[keep] - lo)
        np.testing.assert_array_equal(va, vals[keep])
        np.testing.assert_array_equal(bb, b[lo:hi])
        np.testing.assert_array_equal(cc, c)


def test_partition_rows_respects_rigid_blocks():
    cone = {"z": 3, "l": 40, "q": [50, 7], "s": [4, 3], "ep": 5}
    m = 3 + 40 + 57 + 10 + 6 + 15
    rng = np.random.default_rng(0)
    w = rng.integers(0, 20, size=m)
    for world in (1, 2, 3, 4, 8):
        bnd = native.partition_rows(cone, w, world)
        assert bnd[0] == 0 and bnd[-1] == m and np.all(np.diff(bnd) >= 0)
        rigid = [(100, 110), (110, 116)] + [(116 + 3 * i, 119 + 3 * i) for i in range(5)]
        for cut in bnd[1:-1]:
            assert not any(lo < cut < hi for lo, hi in rigid), (world, cut)


def test_generators_valid_csc():
    for prob in (G.gen_lp("lp_feasible", 20, 40, 0), G.gen_lp("lp_infeasible", 20, 40, 1),
                 G.gen_lp("lp_unbounded", 20, 40, 2), G.gen_lp_soc(300, 100, 0.05, 10, 5, 0),
                 G.gen_cone_mix(n_psd=6, n_exp=4, n_soc=3, l=20, z=2, n=30),
                 G.gen_lasso(20, 8, 60, 0), G.gen_portfolio(30, 4, 0)):
        colptr, rowidx, vals, b, c, cone = prob
        n = colptr.size - 1
        m = b.size
        assert c.size == n
        for j in range(n):
            r = rowidx[colptr[j]:colptr[j + 1]]
            assert np.all(np.diff(r) > 0) and (r.size == 0 or (r[0] >= 0 and r[-1] < m))
        dim = (cone["z"] + cone["l"] + sum(cone["q"]) + sum(k * (k + 1) // 2 for k in cone["s"])
               + 3 * cone["ep"])
        assert dim == m
