"""Load the golden fixtures written by tests/golden/make_golden.py."""

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names(pattern="traj_*.npz"):
    return sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, pattern)))


def load(name):
    z = np.load(os.path.join(GOLDEN, f"traj_{name}.npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["cone"] = json.loads(str(d["cone"]))
    d["settings"] = json.loads(str(d["settings"]))
    d["status"] = str(d["status"])
    d["rowidx"] = d["rowidx"].astype(np.int64)
    for k in ("m", "n", "iterations", "cg_iters"):
        d[k] = int(d[k])
    return d


def known_answers():
    with open(os.path.join(GOLDEN, "known_answers.json")) as fh:
        return json.load(fh)


def cones():
    z = np.load(os.path.join(GOLDEN, "cones.npz"))
    return {k: z[k] for k in z.files}, json.loads(str(z["specs"]))


def eps_tuple(st):
    return (st["eps_pri"], st["eps_dual"], st["eps_gap"], st["eps_infeas"], st["eps_unbdd"])


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)) if b.size else 0.0


def check_golden():
    """Reference checker reports (tests/golden/make_check_golden.py)."""
    z = np.load(os.path.join(GOLDEN, "check_golden.npz"))
    meta = json.loads(str(z["meta"]))
    for rep in meta:
        rep["vecs"] = {k: z[f"{rep['tag']}.{k}"] for k in ("x", "y", "s", "certificate")
                       if f"{rep['tag']}.{k}" in z.files}
    return meta
