"""The native LASSO generator (host_gen.cpp scs_gen_lasso) and its pure-numpy
twin (generators.gen_lasso_hashed) must build the same instance bit for bit:
the CPU reference arm of bench.py and the production-scale golden fixture
(tests/golden/make_c3_golden.py) use the twin, the GPU tests the library."""

import numpy as np
import pytest

from paper_1312_3039_b200 import generators as G
from paper_1312_3039_b200 import native


@pytest.mark.parametrize("p,q,nnz_f,seed", [
    (12, 40, 100, 5),        # sparse columns, few duplicates
    (7, 5, 30, 3),           # dense columns (2k > q): key selection
    (30, 8, 200, 1),         # mixed k, k + 1 per column, dense
    (200, 300, 50_000, 2),   # many duplicate redraw rounds (k/q ~ 0.8)
    (500, 8998, 1_000_000, 1),
])
def test_hashed_twin_bit_identical(p, q, nnz_f, seed):
    a = native.gen_lasso(p, q, nnz_f, seed=seed, threads=3)
    b = G.gen_lasso_hashed(p, q, nnz_f, seed=seed)
    for x, y in zip(a[:5], b[:5]):
        assert x.dtype == y.dtype
        np.testing.assert_array_equal(x, y)
    assert a[5] == b[5]


def test_hashed_distribution():
    """Entries approximately N(0,1) (Irwin-Hall of 4 uniforms), rows distinct
    and sorted per column, nnz exact."""
    p, q, nnz_f = 300, 5000, 300_000
    colptr, rowidx, vals, b, c, cone = G.gen_lasso_hashed(p, q, nnz_f, seed=7)
    f = vals[np.abs(vals) != 1.0] / 2.0
    assert f.size == nnz_f
    assert abs(f.mean()) < 0.01 and abs(f.std() - 1.0) < 0.01
    assert np.abs(f).max() <= 2 * np.sqrt(3.0)
    for j in range(0, p, 37):
        r = rowidx[colptr[j]:colptr[j + 1]]
        assert np.all(np.diff(r) > 0)
