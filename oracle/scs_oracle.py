"""CPU oracle for the SCS indirect-method hot path.

TEST INFRASTRUCTURE ONLY.  This module is a numpy restatement of the
reference algorithm (``conesplit`` 0.1.0 under /root/reference/pkg/src) and
is used exclusively as a *checker*: by ``tests/``, by
``__graft_entry__.smoke()`` and by the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``.  The product path (``paper_1312_3039_b200``) never
imports it; it fails loudly when its CUDA library is missing.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``), including 50-iteration (u, v)
trajectories and final solutions.  The exponential cone is NOT in the
reference: its projection here is an independent restatement of
the standard univariate root formulation and is "parity unpinned" -- it is
checked only through Moreau/KKT properties.

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SQRT2 = math.sqrt(2.0)
JACOBI_REL_TOL = 1e-12      # cones.py:19
JACOBI_MAX_SWEEPS = 100     # cones.py:20
TAU_EXTRACT_THRESHOLD = 1e-8  # solver.py:40
# Timing fidelity (bench.py's CPU reference arm sets it): also compute the
# reference's final exact CG residual (sparse_linalg.py:289), whose value
# solve_kkt discards (embedding.py:110), so the port does the reference's
# full per-iteration work -- 2 more SpMVs per CG solve.  No effect on results.
REFERENCE_WORK = False

STATUS = ("solved", "infeasible", "unbounded", "infeasible_and_unbounded",
          "indeterminate", "max_iters_reached")  # solver.py:43-49


# ---------------------------------------------------------------------------
# sparse products (sparse_linalg.py:121-138): bincount scatter, ascending
# index order per output entry, products rounded before the sum.
# ---------------------------------------------------------------------------
class Csc:
    """CSC view: colptr (n+1), rowidx, vals -- the reference SparseMatrix."""

    def __init__(self, m, n, colptr, rowidx, vals):
        self.m, self.n = int(m), int(n)
        self.colptr = np.ascontiguousarray(colptr, dtype=np.int64)
        self.rowidx = np.ascontiguousarray(rowidx, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        # expanded column of every stored entry (sparse_linalg.py:61-67)
        self.colidx = np.repeat(np.arange(self.n, dtype=np.int64),
                                np.diff(self.colptr))

    @property
    def nnz(self):
        return int(self.vals.size)

    def with_vals(self, vals):
        out = Csc.__new__(Csc)
        out.m, out.n = self.m, self.n
        out.colptr, out.rowidx, out.colidx = self.colptr, self.rowidx, self.colidx
        out.vals = vals
        return out

    def dense(self):
        d = np.zeros((self.m, self.n))
        d[self.rowidx, self.colidx] = self.vals
        return d


def mul(A: Csc, x):
    """y = A x   (sparse_linalg.py:121-128)."""
    if A.nnz == 0:
        return np.zeros(A.m)
    return np.bincount(A.rowidx, weights=A.vals * x[A.colidx], minlength=A.m)


def mul_t(A: Csc, y):
    """x = A^T y (sparse_linalg.py:131-138)."""
    if A.nnz == 0:
        return np.zeros(A.n)
    return np.bincount(A.colidx, weights=A.vals * y[A.rowidx], minlength=A.n)


# ---------------------------------------------------------------------------
# cones (cones.py:89-139 block layout; ep appended after PSD)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Cone:
    z: int = 0
    l: int = 0
    q: tuple = ()
    s: tuple = ()
    ep: int = 0

    @property
    def dim(self):
        return (self.z + self.l + sum(self.q)
                + sum(k * (k + 1) // 2 for k in self.s) + 3 * self.ep)

    def blocks(self):
        """(kind, offset, length, side) in the fixed order (cones.py:121-139)."""
        off = 0
        if self.z:
            yield ("zero", off, self.z, 0)
            off += self.z
        if self.l:
            yield ("nonneg", off, self.l, 0)
            off += self.l
        for d in self.q:
            yield ("soc", off, d, 0)
            off += d
        for k in self.s:
            yield ("psd", off, k * (k + 1) // 2, k)
            off += k * (k + 1) // 2
        for _ in range(self.ep):
            yield ("exp", off, 3, 0)
            off += 3


def cone_from_spec(spec) -> Cone:
    """Accept a reference ConeSpec, a dict {"z","l","q","s"[,"ep"]} or a Cone."""
    if isinstance(spec, Cone):
        return spec
    if isinstance(spec, dict):
        return Cone(int(spec.get("z", 0)), int(spec.get("l", 0)),
                    tuple(int(v) for v in spec.get("q", ())),
                    tuple(int(v) for v in spec.get("s", ())),
                    int(spec.get("ep", 0)))
    return Cone(int(spec.zero_dim), int(spec.nonneg_dim),
                tuple(int(v) for v in spec.soc_dims),
                tuple(int(v) for v in spec.psd_sides),
                int(getattr(spec, "exp_dim", 0)))


def _tril_index(side):
    """Column-major lower triangle (rows, cols, scale) (cones.py:31-40)."""
    cols = np.repeat(np.arange(side), np.arange(side, 0, -1))
    rows = np.concatenate([np.arange(j, side) for j in range(side)])
    return rows, cols, np.where(rows == cols, 1.0, SQRT2)


def svec_to_mat(vec, side):
    """cones.py:53-64."""
    rows, cols, scale = _tril_index(side)
    mat = np.zeros((side, side))
    mat[rows, cols] = vec / scale
    mat[cols, rows] = mat[rows, cols]
    return mat


def mat_to_svec(mat):
    """cones.py:43-50."""
    rows, cols, scale = _tril_index(mat.shape[0])
    return mat[rows, cols] * scale


def jacobi(a, rel_tol=JACOBI_REL_TOL, max_sweeps=JACOBI_MAX_SWEEPS):
    """Cyclic Jacobi eigendecomposition (_kernels.py:119-191).

    Returns (eigenvalues, eigenvectors, sweeps) with sweeps == -1 on failure.
    Pure Python: only used on the small blocks of the tests.
    """
    n = a.shape[0]
    M = [list(map(float, row)) for row in a]
    V = [[1.0 if i == j else 0.0 for j in range(n)] for i in range(n)]
    thresh = rel_tol * math.sqrt(sum(v * v for row in M for v in row))
    if n == 1:
        return np.array([M[0][0]]), np.eye(1), 0

    def offnorm():
        return math.sqrt(sum(2.0 * M[i][j] * M[i][j]
                             for i in range(n) for j in range(i + 1, n)))

    for sweep in range(max_sweeps):
        if offnorm() <= thresh:
            return np.array([M[i][i] for i in range(n)]), np.array(V), sweep
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = M[p][q]
                if apq == 0.0:
                    continue
                app, aqq = M[p][p], M[q][q]
                tau = (aqq - app) / (2.0 * apq)
                root = math.sqrt(1.0 + tau * tau)
                t = 1.0 / (tau + root) if tau >= 0.0 else 1.0 / (tau - root)
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                M[p][p] = app - t * apq
                M[q][q] = aqq + t * apq
                M[p][q] = M[q][p] = 0.0
                for k in range(n):
                    if k != p and k != q:
                        akp, akq = M[k][p], M[k][q]
                        M[k][p] = M[p][k] = c * akp - s * akq
                        M[k][q] = M[q][k] = s * akp + c * akq
                for k in range(n):
                    vkp, vkq = V[k][p], V[k][q]
                    V[k][p] = c * vkp - s * vkq
                    V[k][q] = s * vkp + c * vkq
    if offnorm() <= thresh:
        return np.array([M[i][i] for i in range(n)]), np.array(V), max_sweeps
    return np.zeros(n), np.array(V), -1


def proj_soc(blk):
    """Second-order cone (cones.py:172-184)."""
    t, z = blk[0], blk[1:]
    nz = math.sqrt(float(z @ z))
    if nz <= -t:
        return np.zeros_like(blk)
    if nz <= t:
        return blk.copy()
    a = 0.5 * (nz + t)
    out = np.empty_like(blk)
    out[0] = a
    out[1:] = (a / nz) * z
    return out


def proj_psd(blk, side):
    """PSD cone via Jacobi eig and eigenvalue clamp (cones.py:147-191)."""
    mat = svec_to_mat(blk, side)
    sym = 0.5 * (mat + mat.T)
    vals, vecs, sweeps = jacobi(sym)
    if sweeps < 0:
        raise RuntimeError("Jacobi eigensolver did not converge")
    order = np.argsort(vals, kind="stable")          # cones.py:168-169
    vals, vecs = vals[order], vecs[:, order]
    return mat_to_svec((vecs * np.maximum(vals, 0.0)) @ vecs.T)


# --- exponential cone: NO reference -- parity unpinned ---------
def _exp_in_primal(r, s, t):
    if s > 0:
        return r / s < 700 and s * math.exp(r / s) <= t
    return r <= 0 and s == 0 and t >= 0


def _exp_in_dual(u, v, w):
    if u < 0:
        return v / u < 700 and -u * math.exp(v / u) <= math.e * w
    return u == 0 and v >= 0 and w >= 0


def _exp_sign(rho, r0, s0, t0):
    """sign(F(rho)) without overflow: F q e^-rho (rho >= 0), F q e^rho (rho < 0)."""
    q = rho * rho - rho + 1.0
    a, b = (rho - 1.0) * r0 + s0, r0 - rho * s0
    if rho >= 0:
        e = math.exp(-rho)
        return a - b * e * e - t0 * q * e
    e = math.exp(rho)
    return a * e * e - b - t0 * q * e


def proj_exp_primal(v0):
    """Projection onto K_exp = cl{(r,s,t): s>0, s exp(r/s) <= t}.

    Hard case: the projection is s*(rho, 1, e^rho) with polar part
    -lam*(-1, rho-1, e^-rho); eliminating s, lam leaves the univariate root
    F(rho) = ((rho-1) r0 + s0) e^rho - (r0 - rho s0) e^-rho - t0 (rho^2 - rho + 1)
    on the interval where s > 0 and lam > 0, found by bisection on an
    overflow-free rescaling of F; t is recovered as t0 + lam e^-rho when
    rho > 0 (s e^rho would amplify the rounding of s by e^rho).
    """
    r0, s0, t0 = (float(x) for x in v0)
    if _exp_in_primal(r0, s0, t0):
        return np.array([r0, s0, t0])
    if _exp_in_dual(-r0, -s0, -t0):
        return np.zeros(3)
    if r0 <= 0 and s0 <= 0:
        return np.array([r0, 0.0, max(t0, 0.0)])
    lo, hi = -math.inf, math.inf
    if r0 > 0:
        lo = max(lo, 1.0 - s0 / r0)
    elif r0 < 0:
        hi = min(hi, 1.0 - s0 / r0)
    if s0 > 0:
        hi = min(hi, r0 / s0)
    elif s0 < 0:
        lo = max(lo, r0 / s0)
    if not math.isfinite(lo):
        lo = (hi if math.isfinite(hi) else 0.0) - 1.0
        while _exp_sign(lo, r0, s0, t0) > 0:
            lo = 2.0 * lo - 1.0
    if not math.isfinite(hi):
        hi = lo + 1.0
        while _exp_sign(hi, r0, s0, t0) < 0:
            hi = 2.0 * abs(hi) + 1.0
    for _ in range(400):
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            break
        if _exp_sign(mid, r0, s0, t0) < 0:
            lo = mid
        else:
            hi = mid
    rho = 0.5 * (lo + hi)
    q = rho * rho - rho + 1.0
    s = ((rho - 1.0) * r0 + s0) / q
    lam = (r0 - rho * s0) / q
    t = t0 + lam * math.exp(-rho) if rho > 0 else s * math.exp(rho)
    return np.array([s * rho, s, t])


def proj_exp_dual(v):
    """Pi_{K*}(v) = v + Pi_K(-v) (Moreau)."""
    return v + proj_exp_primal(-v)


def proj_dual_cone(x, cone: Cone):
    """Projection onto K* (cones.py:220-238); zero block is free."""
    if not np.all(np.isfinite(x)):
        raise ValueError("project_dual_cone: non-finite input")  # cones.py:194-200
    out = np.empty_like(x)
    for kind, off, ln, side in cone.blocks():
        blk = x[off:off + ln]
        if kind == "zero":
            out[off:off + ln] = blk
        elif kind == "nonneg":
            out[off:off + ln] = np.maximum(blk, 0.0)
        elif kind == "soc":
            out[off:off + ln] = proj_soc(blk)
        elif kind == "psd":
            out[off:off + ln] = proj_psd(blk, side)
        else:
            out[off:off + ln] = proj_exp_dual(blk)
    return out


def proj_primal_cone(x, cone: Cone):
    """Projection onto K (cones.py:203-217); zero block maps to 0."""
    out = np.empty_like(x)
    for kind, off, ln, side in cone.blocks():
        blk = x[off:off + ln]
        if kind == "zero":
            out[off:off + ln] = 0.0
        elif kind == "nonneg":
            out[off:off + ln] = np.maximum(blk, 0.0)
        elif kind == "soc":
            out[off:off + ln] = proj_soc(blk)
        elif kind == "psd":
            out[off:off + ln] = proj_psd(blk, side)
        else:
            out[off:off + ln] = proj_exp_primal(blk)
    return out


def proj_embedding(u, n, cone: Cone):
    """R^n x K* x R_+ (cones.py:241-249)."""
    if not np.all(np.isfinite(u)):
        raise ValueError("project_embedding_cone: non-finite input")
    m = cone.dim
    out = np.empty_like(u)
    out[:n] = u[:n]
    out[n:n + m] = proj_dual_cone(u[n:n + m], cone)
    out[-1] = max(u[-1], 0.0)
    return out


# ---------------------------------------------------------------------------
# equilibration and residuals (scaling.py:62-207)
# ---------------------------------------------------------------------------
def row_blocks(cone: Cone):
    """Per-row block id; zero/nonneg rows are singletons (scaling.py:62-71)."""
    sizes = []
    for kind, _off, ln, _side in cone.blocks():
        if kind in ("zero", "nonneg"):
            sizes.extend([1] * ln)
        else:
            sizes.append(ln)
    sizes = np.asarray(sizes, dtype=np.int64)
    return np.repeat(np.arange(sizes.size), sizes), sizes


def _inv_sqrt_or_one(v):
    return np.where(v > 0, 1.0 / np.sqrt(np.where(v > 0, v, 1.0)), 1.0)


def equilibrate(A: Csc, b, c, cone: Cone, sweeps=10):
    """Ruiz-style sweeps then sigma/rho (scaling.py:79-129).

    Returns (A_hat, b_hat, c_hat, D, E, sigma, rho).
    """
    m, n = A.m, A.n
    D, E = np.ones(m), np.ones(n)
    v = A.vals.copy()
    rb, rsz = row_blocks(cone)
    for _ in range(int(sweeps)):
        cs = _inv_sqrt_or_one(np.sqrt(np.bincount(A.colidx, v * v, minlength=n)))
        v *= cs[A.colidx]
        E *= cs
        rn = np.sqrt(np.bincount(A.rowidx, v * v, minlength=m))
        means = np.bincount(rb, rn, minlength=rsz.size) / rsz
        rs = _inv_sqrt_or_one(means[rb])
        v *= rs[A.rowidx]
        D *= rs
    cn = np.sqrt(np.bincount(A.colidx, v * v, minlength=n))
    mean_col = cn[cn > 0].mean() if np.any(cn > 0) else 1.0
    rn = np.sqrt(np.bincount(A.rowidx, v * v, minlength=m))
    means = np.bincount(rb, rn, minlength=rsz.size) / rsz
    mean_row = means[means > 0].mean() if np.any(means > 0) else 1.0
    dbn = np.linalg.norm(D * b)
    ecn = np.linalg.norm(E * c)
    sigma = mean_col / dbn if dbn > 0 else 1.0
    rho = mean_row / ecn if ecn > 0 else 1.0
    return A.with_vals(v), sigma * D * b, rho * E * c, D, E, sigma, rho


@dataclass
class Res:
    """scaling.py:37-55 field order."""
    pri_norm: float
    dual_norm: float
    gap: float
    pri_thresh: float
    dual_thresh: float
    gap_thresh: float
    unbdd_measure: float
    infeas_measure: float


def residuals(u, v, A: Csc, b, c, D, E, sigma, rho):
    """Original-units residuals from scaled iterates (scaling.py:148-207)."""
    n, m = A.n, A.m
    ux, uy, ut = u[:n], u[n:n + m], u[-1]
    vs = v[n:n + m]
    Di, Ei = 1.0 / D, 1.0 / E
    Aux = mul(A, ux)
    Atuy = mul_t(A, uy)
    bn = np.linalg.norm(Di * b) / sigma
    cn = np.linalg.norm(Ei * c) / rho
    cux, buy = float(c @ ux), float(b @ uy)
    cref = np.linalg.norm(Ei * c) or 1.0
    bref = np.linalg.norm(Di * b) or 1.0
    unbdd = np.linalg.norm(Di * (Aux + vs)) * cref / (-cux) if cux < 0 else np.inf
    infeas = np.linalg.norm(Ei * Atuy) * bref / (-buy) if buy < 0 else np.inf
    if ut > 0:
        pri = np.linalg.norm(Di * ((Aux + vs) / ut - b)) / sigma
        dual = np.linalg.norm(Ei * (Atuy / ut + c)) / rho
        ctx = cux / ut / (rho * sigma)
        bty = buy / ut / (rho * sigma)
        gap, gth = ctx + bty, 1.0 + abs(ctx) + abs(bty)
    else:
        pri = dual = gap = np.inf
        gth = 1.0
    return Res(pri, dual, gap, 1.0 + bn, 1.0 + cn, gth, unbdd, infeas)


def termination(res: Res, eps):
    """solver.py:210-234; eps = (pri, dual, gap, infeas, unbdd)."""
    if (res.pri_norm <= eps[0] * res.pri_thresh and
            res.dual_norm <= eps[1] * res.dual_thresh and
            abs(res.gap) <= eps[2] * res.gap_thresh):
        return "solved"
    inf = res.infeas_measure <= eps[3]
    unb = res.unbdd_measure <= eps[4]
    if inf and unb:
        return "infeasible_and_unbounded"
    if inf:
        return "infeasible"
    if unb:
        return "unbounded"
    return None


# ---------------------------------------------------------------------------
# linear system: CG on I + A^T A (sparse_linalg.py:253-290, embedding.py:86-197)
# ---------------------------------------------------------------------------
def cg(A: Csc, rhs, x0, tol, max_iter, minv=None):
    """Plain warm-started CG; returns (x, iterations).

    The reference's final exact residual (sparse_linalg.py:289) is dropped by
    its only caller (embedding.py:110) and is computed here only when
    REFERENCE_WORK is set (timing fidelity).
    ``minv`` (opt-in, not in the reference -- parity unpinned): Jacobi
    preconditioner, p = M^-1 r, alpha/beta from r'M^-1 r; the stopping test
    stays on ||r|| as in the reference.
    """
    if tol <= 0:
        raise ValueError("cg_solve: tol must be positive")

    def gram(v):
        return v + mul_t(A, mul(A, v))

    x = np.array(x0, dtype=float, copy=True)
    r = rhs - gram(x)
    res = np.linalg.norm(r)
    if not np.isfinite(res):
        raise ValueError("cg_solve: non-finite residual")
    if res <= tol:
        return x, 0
    if minv is None:
        p = r.copy()
        rs = res * res
    else:
        p = minv * r
        rs = r @ p
    it = 0
    for _ in range(max_iter):
        Gp = gram(p)
        den = p @ Gp
        if not np.isfinite(den) or den <= 0:
            raise ValueError("cg_solve: operator is not positive definite on iterates")
        a = rs / den
        x += a * p
        r -= a * Gp
        it += 1
        rs_new = r @ r
        if not np.isfinite(rs_new):
            raise ValueError("cg_solve: non-finite residual")
        if np.sqrt(rs_new) <= tol:
            break
        if minv is None:
            p = r + (rs_new / rs) * p
            rs = rs_new
        else:
            z = minv * r
            rz = r @ z
            p = z + (rz / rs) * p
            rs = rz
    if REFERENCE_WORK:
        np.linalg.norm(rhs - gram(x))  # sparse_linalg.py:289, discarded like the reference
    return x, it


class OracleSolver:
    """Workspace restatement, indirect mode only (solver.py:291-378)."""

    def __init__(self, A: Csc, b, c, cone, *, alpha=1.5, max_iters=2500,
                 eps=(1e-3,) * 5, check_interval=1, cg_max=2, cg_tol=None,
                 normalize=True, sweeps=10, precond=False):
        self.cone = cone_from_spec(cone)
        self.A0, self.b0, self.c0 = A, np.asarray(b, float), np.asarray(c, float)
        self.alpha, self.max_iters, self.eps = alpha, max_iters, tuple(eps)
        self.check_interval, self.cg_max, self.cg_tol = check_interval, cg_max, cg_tol
        self.normalize, self.sweeps = normalize, sweeps
        self.precond = precond
        self.cg_iters_total = 0
        self._rescale()
        self.cg_warm = np.zeros(A.n)
        self._refresh()

    def _rescale(self):  # solver.py:318-323
        if self.normalize:
            (self.A, self.b, self.c, self.D, self.E, self.sigma,
             self.rho) = equilibrate(self.A0, self.b0, self.c0, self.cone, self.sweeps)
        else:
            self.A, self.b, self.c = self.A0, self.b0.copy(), self.c0.copy()
            self.D, self.E = np.ones(self.A0.m), np.ones(self.A0.n)
            self.sigma = self.rho = 1.0
        self.minv = None
        if self.precond:  # opt-in Jacobi PCG on diag(I + A^T A)
            colsq = np.bincount(np.repeat(np.arange(self.A.n), np.diff(self.A.colptr)),
                                self.A.vals * self.A.vals, minlength=self.A.n)
            self.minv = 1.0 / (1.0 + colsq)

    def _kkt(self, w, tol, max_iter):
        """solve_kkt indirect branch (embedding.py:101-114)."""
        n = self.A.n
        rhs = w[:n] - mul_t(self.A, w[n:])
        zx, it = cg(self.A, rhs, self.cg_warm, tol, max_iter, self.minv)
        self.cg_warm = zx.copy()
        self.cg_iters_total += it
        return np.concatenate([zx, w[n:] + mul(self.A, zx)])

    def _refresh(self):
        """g = M^-1 h, denom (embedding.py:145-162)."""
        self.h = np.concatenate([self.c, self.b])
        tight = 1e-9 * (1.0 + np.linalg.norm(self.h))
        saved = self.cg_warm
        self.cg_warm = np.zeros(self.A.n)
        self.g = self._kkt(self.h, tight, 10 * self.A.n + 100)
        self.cg_warm = saved
        self.denom = 1.0 + self.h @ self.g
        if self.denom < 1.0 - 1e-9:
            raise RuntimeError(f"Schur denominator {self.denom} below 1")

    def update_vectors(self, b=None, c=None):  # solver.py:325-334
        if b is not None:
            self.b0 = np.asarray(b, float)
        if c is not None:
            self.c0 = np.asarray(c, float)
        self._rescale()
        self._refresh()

    def affine(self, w, k):
        """project_affine with advance_schedule (embedding.py:165-197)."""
        n = self.A.n
        rhs = w[:-1] - w[-1] * self.h
        tol = self.cg_tol if self.cg_tol is not None else \
            1e-3 * (1.0 + np.linalg.norm(rhs)) / k ** 1.5
        p = self._kkt(rhs, tol, self.cg_max)
        corr = (self.h @ p) / self.denom
        uxy = p - corr * self.g
        out = np.empty(w.size)
        out[:-1] = uxy
        out[-1] = w[-1] + self.c @ uxy[:n] + self.b @ uxy[n:]
        return out

    def step(self, u, v, k):
        """iterate_once (solver.py:153-166)."""
        w = u + v
        ut = self.affine(w, k)
        ub = self.alpha * ut + (1.0 - self.alpha) * u
        un = proj_embedding(ub - v, self.A.n, self.cone)
        vn = (v - ub) + un
        return un, vn

    def residuals(self, u, v):
        return residuals(u, v, self.A, self.b, self.c, self.D, self.E,
                         self.sigma, self.rho)

    def solve(self, warm_start=None, on_iteration=None, max_iters=None):
        """Workspace.solve (solver.py:336-378) -> dict."""
        n, m = self.A.n, self.A.m
        max_iters = self.max_iters if max_iters is None else max_iters
        u, v = np.zeros(n + m + 1), np.zeros(n + m + 1)
        u[-1] = 1.0
        if warm_start is None:
            v[-1] = 1.0
        else:  # solver.py:345-348, scaling.py:132-137, solver.py:140-149
            x0, y0, s0 = (np.asarray(t, float) for t in warm_start)
            u[:n] = self.sigma * x0 / self.E
            u[n:n + m] = self.rho * y0 / self.D
            v[n:n + m] = self.sigma * self.D * s0
        self.cg_warm = np.zeros(n)  # reset_schedule (embedding.py:45-48)
        status, res, it = None, None, 0
        while it < max_iters:
            it += 1
            u, v = self.step(u, v, it)
            if on_iteration is not None:
                on_iteration(it, u, v)
            if it % self.check_interval == 0:
                res = self.residuals(u, v)
                status = termination(res, self.eps)
                if status is not None:
                    break
        if status is None:
            res = self.residuals(u, v)
            status = ("max_iters_reached"
                      if u[-1] > TAU_EXTRACT_THRESHOLD * np.linalg.norm(u)
                      else "indeterminate")
        out = extract(u, v, status, self.D, self.E, self.sigma, self.rho,
                      self.A0, self.b0, self.c0)
        out.update(iterations=it, residuals=res, u=u, v=v,
                   cg_iters=self.cg_iters_total)
        return out


def extract(u, v, status, D, E, sigma, rho, A0: Csc, b0, c0):
    """extract_solution + _point_residuals (solver.py:237-288)."""
    n, m = A0.n, A0.m
    ux, uy, ut, vs = u[:n], u[n:n + m], u[-1], v[n:n + m]
    out = dict(status=status, x=None, y=None, s=None, certificate=None,
               certificate_unbounded=None, primal_obj=np.nan, dual_obj=np.nan,
               pri_res=np.nan, dual_res=np.nan, gap=np.nan)
    if status in ("solved", "max_iters_reached"):
        x = E * (ux / ut) / sigma
        s = (vs / ut) / (D * sigma)
        y = D * (uy / ut) / rho
        out.update(x=x, y=y, s=s, primal_obj=c0 @ x, dual_obj=-(b0 @ y))
        out["pri_res"] = np.linalg.norm(mul(A0, x) + s - b0) / (1.0 + np.linalg.norm(b0))
        out["dual_res"] = np.linalg.norm(mul_t(A0, y) + c0) / (1.0 + np.linalg.norm(c0))
        ctx, bty = c0 @ x, b0 @ y
        out["gap"] = abs(ctx + bty) / (1.0 + abs(ctx) + abs(bty))
    if status in ("infeasible", "infeasible_and_unbounded"):
        yd = D * uy / rho
        out.update(certificate=yd / (-(b0 @ yd)), primal_obj=np.inf, dual_obj=np.inf)
    if status in ("unbounded", "infeasible_and_unbounded"):
        xd = E * ux / sigma
        ray = xd / (-(c0 @ xd))
        if status == "unbounded":
            out.update(certificate=ray, primal_obj=-np.inf, dual_obj=-np.inf)
        else:
            out["certificate_unbounded"] = ray
    return out
