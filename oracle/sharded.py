"""Row-sharded restatement of the oracle (TEST INFRASTRUCTURE ONLY).

The same algorithm as ``scs_oracle.OracleSolver`` with A split by rows over
`world` ranks, written exactly along the decomposition the CUDA path uses
(DESIGN.md §7): n-length vectors and CG replicated; m-length
vectors sharded; all-reduces of the A^T partial products, of every y-part
scalar, of equilibration column sums / block-row sums, and of the partial
norms (and head entries) of second-order cones that straddle a bound.
``allreduce(array) -> array`` is supplied by the caller (gloo in the tests),
so this checks the decomposition on CPU, independent of any GPU.
"""

from __future__ import annotations

import math

import numpy as np

from . import scs_oracle as O


class ShardedOracle:
    def __init__(self, A_local: O.Csc, b_local, c, cone, row_lo, m_global, allreduce, *,
                 alpha=1.5, eps=(1e-3,) * 5, cg_max=2, sweeps=10):
        self.A0 = A_local
        self.b0, self.c0 = np.asarray(b_local, float), np.asarray(c, float)
        self.cone = O.cone_from_spec(cone)
        self.lo, self.M = int(row_lo), int(m_global)
        self.hi = self.lo + A_local.m
        self.ar = allreduce
        self.alpha, self.eps, self.cg_max, self.sweeps = alpha, eps, cg_max, sweeps
        self._blocks()
        self._equilibrate()
        self._g()

    # -- layout -------------------------------------------------------------
    def _blocks(self):
        """Global blocks clipped to [lo, hi): (kind, global off, length, side)."""
        self.local = []
        self.segs = []        # non-singleton blocks: (global id, local a, local b, global len)
        gid = 0
        for kind, off, ln, side in self.cone.blocks():
            a, b = max(off, self.lo), min(off + ln, self.hi)
            if kind in ("soc", "psd", "exp"):
                if b > a:
                    self.segs.append((gid, a - self.lo, b - self.lo, ln))
                gid += 1
            if b > a:
                self.local.append((kind, off, ln, side, a - self.lo, b - self.lo))
        self.nseg = gid
        self.glen = np.array([ln for kind, _, ln, _ in self.cone.blocks()
                              if kind in ("soc", "psd", "exp")], float)

    # -- helpers ---------------------------------------------------------------
    def mul(self, x):
        return O.mul(self.A, x)

    def mul_t(self, y):
        return self.ar(O.mul_t(self.A, y))

    def ydot(self, a, b):
        return float(self.ar(np.array([a @ b]))[0])

    # -- equilibration (scaling.py:79-129) --------------------------------------
    def _row_scale(self, rn):
        """Block means of row norms over the global blocks (scaling.py:74-112)."""
        sums = np.zeros(self.nseg)
        for gid, a, b, _ in self.segs:
            sums[gid] = rn[a:b].sum()
        sums = self.ar(sums)
        means = sums / self.glen
        target = rn.copy()
        for gid, a, b, _ in self.segs:
            target[a:b] = means[gid]
        return O._inv_sqrt_or_one(target), means

    def _equilibrate(self):
        A, m, n = self.A0, self.A0.m, self.A0.n
        v = A.vals.copy()
        D, E = np.ones(m), np.ones(n)
        for _ in range(self.sweeps):
            cn = np.sqrt(self.ar(np.bincount(A.colidx, v * v, minlength=n)))
            cs = O._inv_sqrt_or_one(cn)
            v *= cs[A.colidx]
            E *= cs
            rn = np.sqrt(np.bincount(A.rowidx, v * v, minlength=m))
            rs, _ = self._row_scale(rn)
            v *= rs[A.rowidx]
            D *= rs
        cn = np.sqrt(self.ar(np.bincount(A.colidx, v * v, minlength=n)))
        mean_col = cn[cn > 0].mean() if np.any(cn > 0) else 1.0
        rn = np.sqrt(np.bincount(A.rowidx, v * v, minlength=m))
        _, means = self._row_scale(rn)
        single = np.ones(m, bool)
        for _, a, b, _ in self.segs:
            single[a:b] = False
        s1 = rn[single & (rn > 0)]
        sc = self.ar(np.array([s1.sum(), float(s1.size)]))
        mp = means[means > 0]
        tot, cnt = sc[0] + mp.sum(), sc[1] + mp.size
        mean_row = tot / cnt if cnt > 0 else 1.0
        dbn = math.sqrt(self.ydot(D * self.b0, D * self.b0))
        ecn = np.linalg.norm(E * self.c0)
        self.sigma = mean_col / dbn if dbn > 0 else 1.0
        self.rho = mean_row / ecn if ecn > 0 else 1.0
        self.A = A.with_vals(v)
        self.D, self.E = D, E
        self.b = self.sigma * D * self.b0
        self.c = self.rho * E * self.c0

    # -- linear system ----------------------------------------------------------
    def _cg(self, rhs, x0, tol, cap):
        def gram(p):
            return p + self.mul_t(self.mul(p))
        x = x0.copy()
        r = rhs - gram(x)
        res = np.linalg.norm(r)
        if res <= tol:
            return x, 0
        p, rs, it = r.copy(), res * res, 0
        for _ in range(cap):
            Gp = gram(p)
            a = rs / (p @ Gp)
            x += a * p
            r -= a * Gp
            it += 1
            rn = r @ r
            if math.sqrt(rn) <= tol:
                break
            p = r + (rn / rs) * p
            rs = rn
        return x, it

    def _kkt(self, wx, wy, x0, tol, cap):
        rhs = wx - self.mul_t(wy)
        zx, _ = self._cg(rhs, x0, tol, cap)
        return zx, wy + self.mul(zx)

    def _g(self):
        hn = math.sqrt(self.c @ self.c + self.ydot(self.b, self.b))
        n = self.A.n
        self.gx, self.gy = self._kkt(self.c, self.b, np.zeros(n), 1e-9 * (1 + hn), 10 * n + 100)
        self.denom = 1.0 + self.c @ self.gx + self.ydot(self.b, self.gy)

    # -- cone step (cones.py:220-249) -------------------------------------------
    def _project(self, t):
        out = np.empty_like(t)
        soc_parts = {}
        for kind, off, ln, side, a, b in self.local:
            blk = t[a:b]
            if kind == "zero":
                out[a:b] = blk
            elif kind == "nonneg":
                out[a:b] = np.maximum(blk, 0.0)
            elif kind == "psd":
                out[a:b] = O.proj_psd(blk, side)
            elif kind == "exp":
                out[a:b] = O.proj_exp_dual(blk)
            else:
                head_local = off >= self.lo
                z = blk[1:] if head_local else blk
                soc_parts[off] = (z @ z, blk[0] if head_local else 0.0)
        # all-reduce partial norms and heads of every SOC (global order)
        socs = [off for kind, off, ln, side in self.cone.blocks() if kind == "soc"]
        buf = np.zeros(2 * len(socs))
        for i, off in enumerate(socs):
            if off in soc_parts:
                buf[2 * i], buf[2 * i + 1] = soc_parts[off]
        buf = self.ar(buf)
        for i, off in enumerate(socs):
            ent = [e for e in self.local if e[0] == "soc" and e[1] == off]
            if not ent:
                continue
            _, off_, ln, _, a, b = ent[0]
            nz, t0 = math.sqrt(buf[2 * i]), buf[2 * i + 1]
            blk = t[a:b]
            if nz <= -t0:
                out[a:b] = 0.0
            elif nz <= t0:
                out[a:b] = blk
            else:
                al = 0.5 * (nz + t0)
                out[a:b] = (al / nz) * blk
                if off_ >= self.lo:
                    out[a] = al
        return out

    # -- iteration ---------------------------------------------------------------
    def solve(self, iters):
        n, m = self.A.n, self.A.m
        ux, uy, ut = np.zeros(n), np.zeros(m), 1.0
        vx, vy, vt = np.zeros(n), np.zeros(m), 1.0
        xw = np.zeros(n)
        traj = []
        for k in range(1, iters + 1):
            wx, wy, wt = ux + vx, uy + vy, ut + vt
            rx, ry = wx - wt * self.c, wy - wt * self.b
            nrm = math.sqrt(rx @ rx + self.ydot(ry, ry))
            tol = 1e-3 * (1.0 + nrm) / k ** 1.5
            px, py = self._kkt(rx, ry, xw, tol, self.cg_max)
            xw = px.copy()
            corr = (self.c @ px + self.ydot(self.b, py)) / self.denom
            tx, ty = px - corr * self.gx, py - corr * self.gy
            tt = (wt + self.c @ tx) + self.ydot(self.b, ty)
            al = self.alpha
            bx, by, bt = al * tx + (1 - al) * ux, al * ty + (1 - al) * uy, al * tt + (1 - al) * ut
            nux, nuy, nut = bx - vx, self._project(by - vy), max(bt - vt, 0.0)
            vx, vy, vt = (vx - bx) + nux, (vy - by) + nuy, (vt - bt) + nut
            ux, uy, ut = nux, nuy, nut
            traj.append((ux.copy(), uy.copy(), ut))
        return traj
