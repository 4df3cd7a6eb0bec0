"""CPU restatement of the reference's independent checker (TEST
INFRASTRUCTURE ONLY): cli.py:163-285 (`conesplit check`), checked against
the reference's own reports in tests/golden/check_golden.npz, and used as
the checker of the device checker (paper_1312_3039_b200/check.py) for the
exponential cone, which the reference does not have."""

from __future__ import annotations

import numpy as np

from . import scs_oracle as O


def membership_margins(vec, cone, dual):
    """cli.py:174-199 (+ exp: -distance to K_exp / K_exp*)."""
    out = []
    off = 0
    z, l = cone.get("z", 0), cone.get("l", 0)
    if z:
        if not dual:
            out.append(("zero", -float(np.max(np.abs(vec[off:off + z])))))
        off += z
    if l:
        out.append(("nonneg", float(np.min(vec[off:off + l]))))
        off += l
    for d in cone.get("q", ()):
        blk = vec[off:off + d]
        off += d
        out.append(("soc", float(blk[0] - np.linalg.norm(blk[1:]))))
    for side in cone.get("s", ()):
        ln = side * (side + 1) // 2
        mat = O.svec_to_mat(vec[off:off + ln], side)   # cli.py:163-175 unpacking
        off += ln
        out.append(("psd", float(np.linalg.eigvalsh(mat).min())))
    for _ in range(cone.get("ep", 0)):
        blk = vec[off:off + 3]
        off += 3
        p = O.proj_exp_dual(blk) if dual else O.proj_exp_primal(blk)
        out.append(("exp", -float(np.linalg.norm(blk - p))))
    return out


def _margins(rows, vec, cone, dual, eps, name):
    floor = -eps * (1.0 + np.linalg.norm(vec))
    ok = True
    for label, margin in membership_margins(vec, cone, dual):
        good = margin >= floor
        ok &= good
        rows.append((f"{name} {label} margin", margin, good))
    return ok


def check(A: O.Csc, b, c, cone, status, eps, x=None, y=None, s=None, certificate=None):
    """(ok, rows) as the reference prints them (cli.py:202-268)."""
    rows = []
    if status in ("solved", "max_iters_reached"):
        pri = np.linalg.norm(O.mul(A, x) + s - b) / (1.0 + np.linalg.norm(b))
        dual = np.linalg.norm(O.mul_t(A, y) + c) / (1.0 + np.linalg.norm(c))
        ctx, bty = c @ x, b @ y
        gap = abs(ctx + bty) / (1.0 + abs(ctx) + abs(bty))
        ok = True
        for label, v in (("primal residual", pri), ("dual residual", dual), ("duality gap", gap)):
            rows.append((label, float(v), v <= eps))
            ok &= v <= eps
        ok &= _margins(rows, s, cone, False, eps, "s")
        ok &= _margins(rows, y, cone, True, eps, "y")
        return bool(ok), rows
    if status in ("infeasible", "infeasible_and_unbounded"):
        resid = float(np.linalg.norm(O.mul_t(A, certificate)))
        bty = float(b @ certificate)
        rows += [("||A^T y|| residual", resid, resid <= eps),
                 ("b^T y + 1", bty + 1.0, abs(bty + 1.0) <= eps)]
        ok = rows[0][2] and rows[1][2]
        ok &= _margins(rows, certificate, cone, True, eps, "y")
        return bool(ok), rows
    ctx = float(c @ certificate)
    rows.append(("c^T x + 1", ctx + 1.0, abs(ctx + 1.0) <= eps))
    ok = rows[0][2]
    ok &= _margins(rows, -O.mul(A, certificate), cone, False, eps, "-Ax")
    return bool(ok), rows
