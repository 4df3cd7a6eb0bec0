"""Is a fixture's final status reproducible by the reference itself under
1-ulp noise?  Runs conesplit on the `mixed_nonorm_cgtol` fixture problem with
every SpMV output perturbed by +-1 ulp (build container only; reads
/root/reference).  Measured: clean -> indeterminate; 6 noisy runs ->
indeterminate x3, max_iters_reached x3 (the divergent trajectory's tau at
max_iters straddles the 1e-8 ||u|| rule of solver.py:366), which is why
tests/test_gpu_parity.py accepts either post-loop status for this fixture."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import conesplit as ref  # noqa: E402
from conesplit import embedding as remb, scaling as rsc, solver as rsolver  # noqa: E402
from conesplit import sparse_linalg as rsl  # noqa: E402

import make_golden as M  # noqa: E402
from paper_1312_3039_b200 import generators as gen  # noqa: E402

mix = gen.gen_planted(dict(z=4, l=30, q=[5, 5, 9], s=[2, 3, 4, 5]), 25, 0.25, 7)
data = M.to_ref(*mix)
st = ref.Settings(linsys_mode="indirect", normalize=False, cg_tol=1e-7)
print("clean", ref.Workspace(data, st).solve().status.value)
spmv0, spmvt0 = rsl.spmv, rsl.spmv_t
rng = np.random.default_rng(0)


def nz(y):
    return y * (1.0 + rng.choice([-1.0, 1.0], size=y.shape) * 2.0 ** -52)


for mod in (remb, rsc, rsolver):
    mod.spmv = lambda A, x: nz(spmv0(A, x))
    mod.spmv_t = lambda A, y: nz(spmvt0(A, y))
for trial in range(6):
    sol = ref.Workspace(data, st).solve()
    print("noisy", trial, sol.status.value, sol.info.iterations)
