"""Independent solution checker -- the checks of the
reference's ``conesplit check`` (cli.py:163-285) with the O(nnz) products
and the per-block cone margins (incl. PSD eigenvalues) on the device.

    ok, rows = check_solution(data, sol, eps=1e-6)

``rows`` is a list of (label, value, ok) in the reference's report order;
``verbose=True`` prints them in the reference's format.  Residuals and cone
memberships are recomputed from the problem data and the returned vectors
only; no solver state is reused (cli.py:158-160).
"""

from __future__ import annotations

import numpy as np

from . import native
from .api import ConeSpec, Status


def _cone_dict(spec: ConeSpec):
    return {"z": spec.zero_dim, "l": spec.nonneg_dim, "q": list(spec.soc_dims),
            "s": list(spec.psd_sides), "ep": getattr(spec, "exp_dim", 0)}


def _labels(spec: ConeSpec, dual: bool):
    out = []
    if spec.zero_dim and not dual:
        out.append("zero")
    if spec.nonneg_dim:
        out.append("nonneg")
    out += ["soc"] * len(spec.soc_dims)
    out += ["psd"] * len(spec.psd_sides)
    out += ["exp"] * getattr(spec, "exp_dim", 0)
    return out


def membership_margins(vec, spec: ConeSpec, dual: bool, device: int = 0):
    """[(label, margin)] per cone block; margin >= 0 (exp: == 0) means
    inside (cli.py:174-199)."""
    m = native.cone_margins(vec, _cone_dict(spec), dual=dual, device=device)
    return list(zip(_labels(spec, dual), (float(v) for v in m)))


def _margin_rows(rows, vec, spec, dual, eps, name, device):
    floor = -eps * (1.0 + np.linalg.norm(vec))
    ok = True
    for label, margin in membership_margins(vec, spec, dual, device):
        good = margin >= floor
        ok &= good
        rows.append((f"{name} {label} margin", margin, good))
    return ok


def check_point(data, sol, eps, device=0):
    """cli.py:202-226."""
    rows = []
    for name, vec, length in (("x", sol.x, data.n), ("y", sol.y, data.m), ("s", sol.s, data.m)):
        if vec is None:
            raise ValueError(f"{name}: missing for a solved-status solution")
        if np.shape(vec) != (length,):
            raise ValueError(f"{name}: expected length {length}, got {np.size(vec)}")
    ax, aty = native.check_products(data.A, x=sol.x, y=sol.y, device=device)
    pri = np.linalg.norm(ax + sol.s - data.b) / (1.0 + np.linalg.norm(data.b))
    dual = np.linalg.norm(aty + data.c) / (1.0 + np.linalg.norm(data.c))
    ct_x = float(data.c @ sol.x)
    bt_y = float(data.b @ sol.y)
    gap = abs(ct_x + bt_y) / (1.0 + abs(ct_x) + abs(bt_y))
    ok = True
    for label, value in (("primal residual", pri), ("dual residual", dual), ("duality gap", gap)):
        good = value <= eps
        ok &= good
        rows.append((label, float(value), good))
    ok &= _margin_rows(rows, sol.s, data.spec, False, eps, "s", device)
    ok &= _margin_rows(rows, sol.y, data.spec, True, eps, "y", device)
    return ok, rows


def check_infeasibility_certificate(data, cert, eps, device=0):
    """cli.py:229-250."""
    if cert is None:
        raise ValueError("certificate: missing for an infeasible-status solution")
    if np.shape(cert) != (data.m,):
        raise ValueError(f"certificate: expected length {data.m}, got {np.size(cert)}")
    _, aty = native.check_products(data.A, y=cert, device=device)
    resid = float(np.linalg.norm(aty))
    bty = float(data.b @ cert)
    rows = [("||A^T y|| residual", resid, resid <= eps), ("b^T y + 1", bty + 1.0,
                                                          abs(bty + 1.0) <= eps)]
    ok = rows[0][2] and rows[1][2]
    ok &= _margin_rows(rows, cert, data.spec, True, eps, "y", device)
    return ok, rows


def check_unboundedness_certificate(data, cert, eps, device=0):
    """cli.py:253-268."""
    if cert is None:
        raise ValueError("certificate: missing for an unbounded-status solution")
    if np.shape(cert) != (data.n,):
        raise ValueError(f"certificate: expected length {data.n}, got {np.size(cert)}")
    ax, _ = native.check_products(data.A, x=cert, device=device)
    ctx = float(data.c @ cert)
    rows = [("c^T x + 1", ctx + 1.0, abs(ctx + 1.0) <= eps)]
    ok = rows[0][2]
    ok &= _margin_rows(rows, -ax, data.spec, False, eps, "-Ax", device)
    return ok, rows


def check_solution(data, sol, eps=1e-6, device=0, verbose=False):
    """Dispatch on the status like cli.py:270-285; returns (ok, rows).
    Indeterminate: nothing to verify -> (True, [])."""
    st = sol.status
    if st in (Status.SOLVED, Status.MAX_ITERS_REACHED):
        ok, rows = check_point(data, sol, eps, device)
    elif st in (Status.INFEASIBLE, Status.INFEASIBLE_AND_UNBOUNDED):
        ok, rows = check_infeasibility_certificate(data, sol.certificate, eps, device)
    elif st is Status.UNBOUNDED:
        ok, rows = check_unboundedness_certificate(data, sol.certificate, eps, device)
    else:
        if verbose:
            print("status=indeterminate: nothing to verify")
        return True, []
    if verbose:
        for label, value, good in rows:
            print(f"{label:<22s} {value: .6e}  [{'ok' if good else 'VIOLATED'}]")
        print(f"check {'passed' if ok else 'FAILED'} at eps={eps:g}")
    return ok, rows
