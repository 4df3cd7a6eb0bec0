"""Golden reports of the reference's independent checker (`conesplit check`,
cli.py:163-285) for the device checker (paper_1312_3039_b200/check.py).

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_check_golden.py

For each fixture problem: solve with the reference (indirect), run the
reference's _check_point / _check_infeasibility_certificate /
_check_unboundedness_certificate at two eps values on the solution and on a
perturbed copy (so VIOLATED rows are covered), and record its printed
(label, value, ok) rows.  Output: check_golden.npz (committed).
"""

import contextlib
import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import conesplit as ref  # noqa: E402
from conesplit import cli as rcli  # noqa: E402
from conesplit import cones as rcones  # noqa: E402
from conesplit import sparse_linalg as rsl  # noqa: E402

from _fixtures import load  # noqa: E402

NAMES = ["tiny_lp", "tiny_infeasible", "tiny_unbounded", "ref_lp_feasible", "ref_lp_infeasible",
         "ref_lp_unbounded", "ref_lasso", "ref_portfolio", "ref_rpca", "mixed"]


def parse(text):
    rows = []
    for line in text.splitlines():
        if "[" not in line:
            continue
        head, flag = line.rsplit("[", 1)
        parts = head.rstrip().rsplit(None, 1)
        rows.append([parts[0].strip(), float(parts[1]), flag.startswith("ok")])
    return rows


def run_check(data, sol, eps):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        st = sol.status
        if st in (ref.Status.SOLVED, ref.Status.MAX_ITERS_REACHED):
            ok = rcli._check_point(data, sol, eps)
        elif st in (ref.Status.INFEASIBLE, ref.Status.INFEASIBLE_AND_UNBOUNDED):
            ok = rcli._check_infeasibility_certificate(data, sol.certificate, eps)
        else:
            ok = rcli._check_unboundedness_certificate(data, sol.certificate, eps)
    return bool(ok), parse(buf.getvalue())


def main():
    out = {}
    meta = []
    rng = np.random.default_rng(5)
    for name in NAMES:
        d = load(name)
        A = rsl.SparseMatrix(d["m"], d["n"], d["colptr"], d["rowidx"], d["vals"])
        cone = d["cone"]
        spec = rcones.ConeSpec(zero_dim=cone.get("z", 0), nonneg_dim=cone.get("l", 0),
                               soc_dims=tuple(cone.get("q", ())),
                               psd_sides=tuple(cone.get("s", ())))
        data = ref.ProblemData(A, d["b"], d["c"], spec)
        st = d["settings"]
        settings = ref.Settings(**{k: st[k] for k in (
            "alpha", "max_iters", "eps_pri", "eps_dual", "eps_gap", "eps_infeas", "eps_unbdd",
            "check_interval", "cg_max", "cg_tol", "normalize", "sweeps")}, linsys_mode="indirect")
        sol = ref.solve(data, settings)
        if sol.status is ref.Status.INDETERMINATE:
            continue
        for variant in ("exact", "perturbed"):
            s2 = sol
            if variant == "perturbed":
                import copy
                s2 = copy.deepcopy(sol)
                for key in ("x", "y", "s", "certificate"):
                    v = getattr(s2, key)
                    if v is not None:
                        setattr(s2, key, v + 1e-3 * rng.standard_normal(v.shape))
            for eps in (1e-3, 1e-6):
                ok, rows = run_check(data, s2, eps)
                tag = f"{name}.{variant}.{eps:g}"
                meta.append({"tag": tag, "name": name, "status": s2.status.value, "eps": eps,
                             "ok": ok, "rows": rows})
                for key in ("x", "y", "s", "certificate"):
                    v = getattr(s2, key)
                    if v is not None:
                        out[f"{tag}.{key}"] = v
    out["meta"] = json.dumps(meta)
    np.savez_compressed(os.path.join(HERE, "check_golden.npz"), **out)
    print(len(meta), "reports")


if __name__ == "__main__":
    main()
