"""Seeded synthetic cone programs (test and benchmark inputs).

These follow the reference generator *encodings* (row/column layout, cone
blocks, planted objects) of ``conesplit.generators``
(/root/reference/pkg/src/conesplit/generators.py) but draw from numpy's
PCG64 so they vectorise; they are NOT bit-compatible with the reference's
pure-Python xoshiro stream (the reference disclaims bit-compatibility too,
rng.py:7-9).  Every function returns ``(colptr, rowidx, vals, b, c, cone)``
with CSC arrays in the reference layout (int64 colptr/rowidx, fp64 vals,
rows strictly increasing per column) and ``cone`` a dict
``{"z","l","q","s","ep"}`` (fileio.py:68-73 plus the exp-cone count).

Huge LASSO instances (1e8-1e9 nnz) come from the multithreaded C generator
``scs_gen_lasso`` in the native library (see ``paper_1312_3039_b200.native``);
``gen_lasso_hashed`` is its bit-identical pure-numpy twin (counter-based
streams), for callers that must not load the native library.
"""

from __future__ import annotations

import math

import numpy as np


def _csc_from_triplets(m, n, rows, cols, vals):
    """Sorted CSC, duplicates summed (sparse_linalg.py:72-97 semantics)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals, np.float64)
    key = cols * m + rows
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    if key.size:
        first = np.ones(key.size, bool)
        first[1:] = key[1:] != key[:-1]
        starts = np.flatnonzero(first)
        vals = np.add.reduceat(vals, starts)
        key = key[starts]
    cols, rows = np.divmod(key, m) if m else (key, key)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
    return colptr, rows.astype(np.int64), vals


def csc_matvec(colptr, rowidx, vals, m, x):
    cols = np.repeat(np.arange(colptr.size - 1), np.diff(colptr))
    return np.bincount(rowidx, weights=vals * x[cols], minlength=m)


def csc_rmatvec(colptr, rowidx, vals, y):
    n = colptr.size - 1
    cols = np.repeat(np.arange(n), np.diff(colptr))
    return np.bincount(cols, weights=vals * y[rowidx], minlength=n)


def _random_columns(rng, m, n, per_col):
    """per_col distinct random rows in every column (generators.py:289-299)."""
    rows = rng.integers(0, m, size=(n, per_col))
    for _ in range(100):
        rows.sort(axis=1)
        dup = np.any(rows[:, 1:] == rows[:, :-1], axis=1)
        if not dup.any():
            break
        rows[dup] = rng.integers(0, m, size=(int(dup.sum()), per_col))
    rows.sort(axis=1)
    cols = np.repeat(np.arange(n), per_col)
    return rows.ravel(), cols, rng.standard_normal(n * per_col)


def gen_lp(kind, n, m, seed):
    """LP over the nonnegative orthant with a planted optimum, Farkas
    certificate or improving ray (generators.py:302-383 recipes)."""
    if not m >= n >= 1:
        raise ValueError("lp families need m >= n >= 1")
    rng = np.random.default_rng(seed)
    per_col = min(m, max(2, round(0.3 * m))) if m <= 60 else 8
    rows, cols, vals = _random_columns(rng, m, n, per_col)
    cone = {"z": 0, "l": m, "q": [], "s": [], "ep": 0}
    if kind == "lp_feasible":
        colptr, ri, va = _csc_from_triplets(m, n, rows, cols, vals)
        x = rng.standard_normal(n)
        tight = rng.permutation(m)[: max(1, m // 2)]
        y = np.zeros(m)
        y[tight] = 0.1 + rng.random(tight.size)
        s = 0.1 + rng.random(m)
        s[tight] = 0.0
        b = csc_matvec(colptr, ri, va, m, x) + s
        c = -csc_rmatvec(colptr, ri, va, y)
        return colptr, ri, va, b, c, cone
    if kind == "lp_infeasible":
        r1 = int(rng.integers(m))
        r2 = int(rng.integers(m - 1))
        r2 += r2 >= r1
        keep = rows != r2
        mir = rows == r1
        rows = np.concatenate([rows[keep], np.full(int(mir.sum()), r2)])
        cols2 = np.concatenate([cols[keep], cols[mir]])
        vals = np.concatenate([vals[keep], -vals[mir]])
        colptr, ri, va = _csc_from_triplets(m, n, rows, cols2, vals)
        b = rng.standard_normal(m)
        b[r2] = -1.0 - b[r1]
        c = -csc_rmatvec(colptr, ri, va, rng.random(m))
        return colptr, ri, va, b, c, cone
    if kind == "lp_unbounded":
        present = np.zeros(m, bool)
        present[rows] = True
        miss = np.flatnonzero(~present)
        rows = np.concatenate([rows, miss])
        cols = np.concatenate([cols, rng.integers(0, n, miss.size)])
        vals = np.concatenate([vals, rng.standard_normal(miss.size)])
        x0 = 0.5 + rng.random(n)
        slack = 0.1 + rng.random(m)
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        reach = np.bincount(rows, weights=vals * x0[cols], minlength=m)
        first = np.searchsorted(rows, np.arange(m))
        vals[first] -= (reach + slack) / x0[cols[first]]
        colptr, ri, va = _csc_from_triplets(m, n, rows, cols, vals)
        c = rng.standard_normal(n)
        j = int(rng.integers(n))
        c[j] -= (c @ x0 + 1.0) / x0[j]
        b = rng.random(m)
        return colptr, ri, va, b, c, cone
    raise ValueError(f"unknown LP family kind {kind!r}")


def _planted_blocks(rng, cone):
    """Complementary (s*, y*) per cone block: s in K, y in K*, s'y = 0."""
    m = (cone["z"] + cone["l"] + sum(cone["q"])
         + sum(k * (k + 1) // 2 for k in cone["s"]) + 3 * cone["ep"])
    s = np.zeros(m)
    y = np.zeros(m)
    off = 0
    z = cone["z"]
    y[off:off + z] = rng.standard_normal(z)
    off += z
    ln = cone["l"]
    tight = rng.random(ln) < 0.5
    y[off:off + ln] = np.where(tight, 0.1 + rng.random(ln), 0.0)
    s[off:off + ln] = np.where(tight, 0.0, 0.1 + rng.random(ln))
    off += ln
    for d in cone["q"]:
        if d == 1:
            s[off] = rng.random()
        else:
            u = rng.standard_normal(d - 1)
            u /= np.linalg.norm(u)
            a, bb = 0.5 + rng.random(), 0.5 + rng.random()
            s[off], s[off + 1:off + d] = a, a * u
            y[off], y[off + 1:off + d] = bb, -bb * u
        off += d
    for k in cone["s"]:
        q, _ = np.linalg.qr(rng.standard_normal((k, k)))
        lam = 0.5 + rng.random(k)
        split = rng.random(k) < 0.5
        S = (q * np.where(split, lam, 0.0)) @ q.T
        Y = (q * np.where(split, 0.0, lam)) @ q.T
        rows, cols = np.tril_indices(k)
        order = np.lexsort((rows, cols))  # column-major lower triangle
        rows, cols = rows[order], cols[order]
        scale = np.where(rows == cols, 1.0, math.sqrt(2.0))
        ln2 = k * (k + 1) // 2
        s[off:off + ln2] = S[rows, cols] * scale
        y[off:off + ln2] = Y[rows, cols] * scale
        off += ln2
    for _ in range(cone["ep"]):
        rho = rng.uniform(-1.0, 1.0)
        a, bb = 0.5 + rng.random(), 0.5 + rng.random()
        s[off:off + 3] = a * np.array([rho, 1.0, math.exp(rho)])
        y[off:off + 3] = bb * np.array([-1.0, rho - 1.0, math.exp(-rho)])
        off += 3
    return s, y


def gen_planted(m_cone, n, density, seed, nnz_per_col=None):
    """Feasible cone program with a planted complementary optimum.

    ``m_cone`` is a cone dict; A (m x n) has uniformly random positions at the
    given density (or ``nnz_per_col`` random rows per column) and N(0,1)
    values; b = A x* + s*, c = -A^T y* (generators.py:321-334 extended to
    SOC/PSD/exp blocks).  This is config 1 (LP+SOC) and the C4 cone mix.
    """
    cone = {"z": 0, "l": 0, "q": [], "s": [], "ep": 0}
    cone.update({k: v for k, v in m_cone.items()})
    rng = np.random.default_rng(seed)
    s, y = _planted_blocks(rng, cone)
    m = s.size
    if nnz_per_col is None:
        nnz = max(1, int(round(density * m * n)))
        lin = np.unique(rng.integers(0, m * n, size=int(nnz * 1.02) + 8))
        lin = rng.permutation(lin)[:nnz]
        cols, rows = np.divmod(lin, m)
    else:
        rows, cols, _ = _random_columns(rng, m, n, nnz_per_col)
    vals = rng.standard_normal(rows.size)
    colptr, ri, va = _csc_from_triplets(m, n, rows, cols, vals)
    x = rng.standard_normal(n)
    b = csc_matvec(colptr, ri, va, m, x) + s
    c = -csc_rmatvec(colptr, ri, va, y)
    return colptr, ri, va, b, c, cone


def gen_lp_soc(m=3000, n=1000, density=0.01, n_soc=100, soc_dim=10, seed=0):
    """Config 1: LP+SOC, l = m - n_soc*soc_dim, q = [soc_dim]*n_soc."""
    cone = {"l": m - n_soc * soc_dim, "q": [soc_dim] * n_soc}
    return gen_planted(cone, n, density, seed)


def gen_lasso(p, q, nnz_f, seed, mu=None):
    """Sparse-F LASSO in gen_lasso's standard form (generators.py:81-120).

    F is q x p with ``nnz_f`` N(0,1) entries spread evenly over its columns at
    uniformly random rows; variables (z, t, w): n = 2p+1, m = 2p+q+2,
    cone {l: 2p, q: [q+2]}.
    """
    rng = np.random.default_rng(seed)
    per = np.full(p, nnz_f // p, np.int64)
    per[: nnz_f % p] += 1
    per = np.minimum(per, q)
    fr = []
    for j in range(p):
        fr.append(np.sort(rng.choice(q, int(per[j]), replace=False)))
    frows = np.concatenate(fr) if fr else np.zeros(0, np.int64)
    fcols = np.repeat(np.arange(p), per)
    fvals = rng.standard_normal(frows.size)
    zhat = np.zeros(p)
    sup = rng.choice(p, max(1, p // 10), replace=False)
    zhat[sup] = rng.standard_normal(sup.size)
    g = np.bincount(frows, weights=fvals * zhat[fcols], minlength=q) + \
        rng.standard_normal(q) * math.sqrt(0.1)
    if mu is None:
        mu = 0.1 * np.max(np.abs(np.bincount(fcols, weights=fvals * g[frows], minlength=p)))
    n, m = 2 * p + 1, 2 * p + q + 2
    idx = np.arange(p)
    r0 = 2 * p
    rows = np.concatenate([idx, idx, p + idx, p + idx, [r0, r0 + 1], r0 + 2 + frows])
    cols = np.concatenate([idx, p + idx, idx, p + idx, [2 * p, 2 * p], fcols])
    vals = np.concatenate([np.ones(p), -np.ones(p), -np.ones(p), -np.ones(p),
                           [-1.0, 1.0], 2.0 * fvals])
    b = np.zeros(m)
    b[r0] = b[r0 + 1] = 1.0
    b[r0 + 2:] = 2.0 * g
    c = np.concatenate([np.zeros(p), mu * np.ones(p), [0.5]])
    colptr, ri, va = _csc_from_triplets(m, n, rows, cols, vals)
    return colptr, ri, va, b, c, {"z": 0, "l": 2 * p, "q": [q + 2], "s": [], "ep": 0}


_M64 = (1 << 64) - 1
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _fmix64(z):
    with np.errstate(over="ignore"):
        return _fmix64_(z)


def _fmix64_(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _base_of(seed, dom, j):
    """Stream bases (host_gen.cpp base_of); j an int64 array."""
    c = np.uint64((seed * 0xD1B54A32D192ED03 + dom * 0xA24BAED4963EE407) & _M64)
    with np.errstate(over="ignore"):
        return _fmix64(c + (np.asarray(j, np.int64) + 1).astype(np.uint64) * _GOLD)


def _draw(base, ctr):
    with np.errstate(over="ignore"):
        return _fmix64(base + (np.asarray(ctr).astype(np.uint64) + np.uint64(1)) * _GOLD)


def _normal4(base, i):
    """host_gen.cpp normal4: Irwin-Hall sum of four 32-bit uniforms, unit variance."""
    i = np.asarray(i).astype(np.uint64)
    a = _draw(base, np.uint64(2) * i)
    b = _draw(base, np.uint64(2) * i + np.uint64(1))
    lo = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    u1 = (a >> s32).astype(np.float64) * 2.0 ** -32
    u2 = (a & lo).astype(np.float64) * 2.0 ** -32
    u3 = (b >> s32).astype(np.float64) * 2.0 ** -32
    u4 = (b & lo).astype(np.float64) * 2.0 ** -32
    return (((u1 + u2) + u3) + u4 - 2.0) * 1.7320508075688772


def _hashed_columns(seed, j0, j1, k, q):
    """Rows (sorted, distinct) and values of F columns [j0, j1), k entries
    each: host_gen.cpp f_column, vectorised over columns."""
    js = np.arange(j0, j1, dtype=np.int64)
    br = _base_of(seed, 0, js)[:, None]
    bv = _base_of(seed, 1, js)[:, None]
    if k == 0:
        return np.zeros((js.size, 0), np.int64), np.zeros((js.size, 0))
    if 2 * k > q:
        r = np.arange(q, dtype=np.int64)
        key = _draw(br, np.uint64(1 << 40) + r.astype(np.uint64)[None, :])
        order = np.argsort(key, axis=1, kind="stable")[:, :k]  # ties -> smaller row
        rows = np.sort(order, axis=1)
    else:
        rows = (_draw(br, np.arange(k, dtype=np.uint64)[None, :]) % np.uint64(q)).astype(np.int64)
        rows.sort(axis=1)
        rnd = 1
        while True:
            dup = np.zeros(rows.shape, bool)
            dup[:, 1:] = rows[:, 1:] == rows[:, :-1]
            if not dup.any():
                break
            ci, pi = np.nonzero(dup)
            ctr = (np.uint64(rnd) << np.uint64(32)) | pi.astype(np.uint64)
            rows[ci, pi] = (_draw(br[ci, 0], ctr) % np.uint64(q)).astype(np.int64)
            cols = np.unique(ci)
            rows[cols] = np.sort(rows[cols], axis=1)
            rnd += 1
    vals = _normal4(bv, np.arange(k, dtype=np.uint64)[None, :])
    return rows, vals


def gen_lasso_hashed(p, q, nnz_f, seed=1, chunk=4096):
    """Pure-numpy twin of the native ``scs_gen_lasso`` (host_gen.cpp): the
    same sparse-F LASSO in gen_lasso's encoding (generators.py:81-120), bit
    for bit, from counter-based fmix64 streams and IEEE-exact arithmetic.
    Used where the native library must not be loaded (the CPU reference arm
    of bench.py, fixture generation).  Returns the usual
    ``(colptr, rowidx, vals, b, c, cone)``."""
    if p < 1 or q < 1 or nnz_f < 0 or nnz_f > p * q:
        raise ValueError("gen_lasso_hashed: bad sizes")
    n, m, r0 = 2 * p + 1, 2 * p + q + 2, 2 * p
    kq, kr = divmod(nnz_f, p)
    kcol = np.full(p, kq, np.int64)
    kcol[:kr] += 1
    fptr = np.zeros(p + 1, np.int64)
    np.cumsum(kcol, out=fptr[1:])
    frows = np.empty(nnz_f, np.int64)
    fvals = np.empty(nnz_f, np.float64)
    for lo_, hi_, k in ((0, kr, kq + 1), (kr, p, kq)):
        for j0 in range(lo_, hi_, chunk):
            j1 = min(hi_, j0 + chunk)
            rr, vv = _hashed_columns(seed, j0, j1, int(k), q)
            frows[fptr[j0]:fptr[j1]] = rr.reshape(-1)
            fvals[fptr[j0]:fptr[j1]] = vv.reshape(-1)
    # planted support: the p/10 columns with the smallest (key, column)
    ks = max(1, p // 10)
    key = _draw(_base_of(seed, 2, 0), np.arange(p, dtype=np.uint64))
    support = np.sort(np.argsort(key, kind="stable")[:ks])
    zhat = _normal4(_base_of(seed, 3, 0), np.arange(ks, dtype=np.uint64))
    # g = F zhat (rows accumulated over the support columns in order) + noise
    sel = np.concatenate([np.arange(fptr[j], fptr[j + 1]) for j in support])
    zrep = np.repeat(zhat, kcol[support])
    g = np.bincount(frows[sel], weights=fvals[sel] * zrep, minlength=q)
    g = g + _normal4(_base_of(seed, 4, 0), np.arange(q, dtype=np.uint64)) * math.sqrt(0.1)
    fcols = np.repeat(np.arange(p), kcol)
    ftg = np.bincount(fcols, weights=fvals * g[frows], minlength=p)
    mu = np.max(np.abs(ftg)) * 0.1
    # CSC (host_gen.cpp fill): column j < p: [j, p+j, F rows], column p+j: [j, p+j]
    cnt = np.empty(n, np.int64)
    cnt[:p] = 2 + kcol
    cnt[p:2 * p] = 2
    cnt[2 * p] = 2
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=colptr[1:])
    nnz = int(colptr[-1])
    rowidx = np.empty(nnz, np.int64)
    vals = np.empty(nnz, np.float64)
    idx = np.arange(p, dtype=np.int64)
    s0 = colptr[:p]
    rowidx[s0], vals[s0] = idx, 1.0
    rowidx[s0 + 1], vals[s0 + 1] = p + idx, -1.0
    fpos = np.repeat(s0 + 2 - fptr[:p], kcol) + np.arange(nnz_f)
    rowidx[fpos] = r0 + 2 + frows
    vals[fpos] = 2.0 * fvals
    s1 = colptr[p:2 * p]
    rowidx[s1], vals[s1] = idx, -1.0
    rowidx[s1 + 1], vals[s1 + 1] = p + idx, -1.0
    rowidx[colptr[2 * p]], vals[colptr[2 * p]] = r0, -1.0
    rowidx[colptr[2 * p] + 1], vals[colptr[2 * p] + 1] = r0 + 1, 1.0
    b = np.zeros(m)
    b[r0] = b[r0 + 1] = 1.0
    b[r0 + 2:] = 2.0 * g
    c = np.zeros(n)
    c[p:2 * p] = mu
    c[2 * p] = 0.5
    return colptr, rowidx, vals, b, c, {"z": 0, "l": 2 * p, "q": [q + 2], "s": [], "ep": 0}


def gen_portfolio(p, q, seed, gamma=10.0):
    """Long-only factor-model portfolio SOCP (generators.py:123-194)."""
    rng = np.random.default_rng(seed)
    mu_ret = np.exp(rng.standard_normal(p))
    F = rng.standard_normal((p, q))
    d = 2.0 * rng.random(p)
    n, m = p + 4, 2 * p + q + 9
    t_col, s_col, u_col, v_col = p, p + 1, p + 2, p + 3
    idx = np.arange(p)
    r0 = 1 + p
    r1 = r0 + p + 1
    r2 = r1 + q + 1
    r3 = r2 + 3
    fr, fc = np.nonzero(F.T)
    rows = np.concatenate([np.zeros(p, np.int64), 1 + idx, [r0], r0 + 1 + idx, [r1],
                           r1 + 1 + fr, [r2, r2 + 1, r2 + 2, r3, r3 + 1, r3 + 2]])
    cols = np.concatenate([idx, idx, [u_col], idx, [v_col], fc,
                           [t_col, t_col, u_col, s_col, s_col, v_col]])
    vals = np.concatenate([np.ones(p), -np.ones(p), [-1.0], -np.sqrt(d), [-1.0],
                           -F.T[fr, fc], [-1.0, 1.0, -2.0, -1.0, 1.0, -2.0]])
    b = np.zeros(m)
    b[0] = 1.0
    b[r2] = b[r2 + 1] = b[r3] = b[r3 + 1] = 1.0
    c = np.zeros(n)
    c[:p] = -mu_ret
    c[t_col] = c[s_col] = gamma
    colptr, ri, va = _csc_from_triplets(m, n, rows, cols, vals)
    cone = {"z": 1, "l": p, "q": [p + 1, q + 1, 3, 3], "s": [], "ep": 0}
    return colptr, ri, va, b, c, cone


def gen_cone_mix(n_psd=50, psd_sides=(3, 4, 5, 6, 7, 8), n_exp=50, n_soc=20,
                 soc_dim=6, l=200, z=10, n=400, nnz_per_col=8, seed=0):
    """Config 4 cone mix: zero + nonneg + SOC + many small PSD + exp cones
    with a planted optimum (exp part parity-unpinned)."""
    rng = np.random.default_rng(seed + 1)
    sides = [int(psd_sides[i % len(psd_sides)]) for i in range(n_psd)]
    rng.shuffle(sides)
    cone = {"z": z, "l": l, "q": [soc_dim] * n_soc, "s": sides, "ep": n_exp}
    return gen_planted(cone, n, None, seed, nnz_per_col=nnz_per_col)


def gen_portfolio_c4(p, q, n_exp, group_sides=(2, 3, 4, 5, 6, 7), n_groups=None, seed=0,
                     gamma=10.0, lam=1.0, kappa=1.0):
    """Config 4 (BASELINE.json configs[3]): the reference's long-only factor
    portfolio (gen_portfolio's encoding, generators.py:123-194) extended with

    * log-utility on ``n_exp`` assets: maximise lam * sum log(p z_i) / p
      through (u_i, 1/p, z_i) in K_exp (e^{p u_i} / p <= z_i), objective
      -lam * sum u_i;
    * sector concentration on ``n_groups`` disjoint asset groups of k assets
      (k cycling through ``group_sides``): [[tau_g, z_g^T], [z_g, I_k / p]]
      PSD (side k+1, i.e. p ||z_g||^2 <= tau_g), objective
      + kappa * sum tau_g -- "many small PSD blocks".
    The 1/p constants keep every block on the scale of the weights
    (z ~ 1/p); with O(1) constants the iteration count grows ~p.

    Variables (z: p, t, s, u, v, tau: n_groups, u_exp: n_exp); rows in cone
    order zero, nonneg, SOC (p+1, q+1, 3, 3), PSD, exp.  Not
    reference-comparable beyond the portfolio core (no exp/PSD in the
    reference)."""
    if not p > q >= 1:
        raise ValueError("portfolio needs p > q >= 1")
    rng = np.random.default_rng(seed)
    sides = []
    covered = 0
    while (n_groups is None and covered + group_sides[len(sides) % len(group_sides)] <= p // 2) or \
            (n_groups is not None and len(sides) < n_groups):
        k = group_sides[len(sides) % len(group_sides)]
        if covered + k > p:
            break
        sides.append(k)
        covered += k
    ng = len(sides)
    if n_exp > p:
        raise ValueError("n_exp must be <= p")
    colptr0, ri0, va0, b0, c0, cone0 = gen_portfolio(p, q, seed, gamma)
    m0, n0 = b0.size, colptr0.size - 1
    cols0 = np.repeat(np.arange(n0), np.diff(colptr0))
    perm = rng.permutation(p)
    tau0 = n0
    uexp0 = n0 + ng
    n = n0 + ng + n_exp
    rows, cols, vals = [ri0], [cols0], [va0]
    # PSD blocks: svec of [[tau, z^T], [z, I]] (column-major lower triangle, sqrt2 off-diagonals)
    r = m0
    b_psd = []
    at = 0
    for g, k in enumerate(sides):
        assets = perm[at:at + k]
        at += k
        side = k + 1
        bb = np.zeros(side * (side + 1) // 2)
        e = 0
        for j in range(side):
            for i in range(j, side):
                if i == 0 and j == 0:
                    rows.append([r + e]); cols.append([tau0 + g]); vals.append([-1.0])
                elif j == 0:
                    rows.append([r + e]); cols.append([assets[i - 1]]); vals.append([-math.sqrt(2.0)])
                elif i == j:
                    bb[e] = 1.0 / p
                e += 1
        b_psd.append(bb)
        r += e
    # exp cones (u_i, 1, z_i)
    ex = perm[:n_exp] if n_exp else np.zeros(0, np.int64)
    er = r + 3 * np.arange(n_exp)
    rows += [er, er + 2]
    cols += [uexp0 + np.arange(n_exp), ex]
    vals += [-np.ones(n_exp), -np.ones(n_exp)]
    b_exp = np.zeros(3 * n_exp)
    b_exp[1::3] = 1.0 / p
    m = r + 3 * n_exp
    b = np.concatenate([b0] + b_psd + [b_exp])
    c = np.concatenate([c0, kappa * np.ones(ng), -lam * np.ones(n_exp)])
    colptr, ri, va = _csc_from_triplets(m, n, np.concatenate([np.asarray(x, np.int64) for x in rows]),
                                        np.concatenate([np.asarray(x, np.int64) for x in cols]),
                                        np.concatenate([np.asarray(x, float) for x in vals]))
    cone = dict(cone0)
    cone["s"] = [k + 1 for k in sides]
    cone["ep"] = int(n_exp)
    return colptr, ri, va, b, c, cone
