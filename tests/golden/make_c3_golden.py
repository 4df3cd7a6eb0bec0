"""Production-scale golden fixture: conesplit itself on BASELINE config 3.

Run in the build container only (imports /root/reference/pkg/src, which does
not exist on the GPU box); takes ~15 min of CPU:

    python tests/golden/make_c3_golden.py

Instance: bench.py CONFIGS["c3"] -- the sparse LASSO-as-SOCP in gen_lasso's
encoding (generators.py:81-120) with p = 5e4, q = 899,998, nnz = 1e8, seed 1,
built by ``generators.gen_lasso_hashed`` (bit-identical to the native
``scs_gen_lasso`` the GPU test uses; tests/test_generators.py pins that).

The reference runs ``Workspace.solve`` (solver.py:336-378) for 50 iterations
(max_iters = 50, eps = 1e-3, indirect CG) and the fixture keeps, compactly:
  * norms of u and v after every iteration 1..50 and the reference's
    cumulative CG count (EmbeddingCache.cg_iters_total, embedding.py:112);
  * a seeded sample of 2e4 entries of u and v at k = 1, 2, 5, 10, 20, 50;
  * the eight Residuals values of every termination check (scaling.py:148-207,
    recorded through check_termination, solver.py:359-363);
  * equilibration: sigma, rho and a sample of D, E (scaling.py:79-129);
  * the final status, iteration count and reported residuals/cg_iters.
Output: tests/golden/c3_ref.npz (~1.5 MB).
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import conesplit as ref  # noqa: E402
from conesplit import cones as rcones  # noqa: E402
from conesplit import solver as rsolver  # noqa: E402
from conesplit import sparse_linalg as rsl  # noqa: E402

from paper_1312_3039_b200 import generators as G  # noqa: E402

CFG = dict(p=50_000, q=899_998, nnz=100_000_000, seed=1)  # bench.py CONFIGS["c3"]
SNAP = (1, 2, 5, 10, 20, 50)
NSAMPLE = 20_000
RES_FIELDS = ("pri_norm", "dual_norm", "gap", "pri_thresh", "dual_thresh", "gap_thresh",
              "unbdd_measure", "infeas_measure")  # scaling.py:48-55


def main(out=os.path.join(HERE, "c3_ref.npz"), iters=50):
    p, q = CFG["p"], CFG["q"]
    t0 = time.perf_counter()
    colptr, rowidx, vals, b, c, cone = G.gen_lasso_hashed(p, q, CFG["nnz"] - 4 * p - 2, CFG["seed"])
    m, n = b.size, colptr.size - 1
    print(f"generated m={m} n={n} nnz={rowidx.size} in {time.perf_counter() - t0:.1f}s", flush=True)
    A = rsl.SparseMatrix(m, n, colptr, rowidx, vals)
    spec = rcones.ConeSpec(zero_dim=0, nonneg_dim=cone["l"], soc_dims=tuple(cone["q"]), psd_sides=())
    data = ref.ProblemData(A, b, c, spec)
    st = ref.Settings(linsys_mode="indirect", max_iters=iters, eps_pri=1e-3, eps_dual=1e-3,
                      eps_gap=1e-3)
    t0 = time.perf_counter()
    ws = ref.Workspace(data, st)
    setup_s = time.perf_counter() - t0
    print(f"reference setup {setup_s:.1f}s", flush=True)
    ell = n + m + 1
    rng = np.random.default_rng(20261019)
    idx = np.sort(rng.choice(ell, min(ell, NSAMPLE), replace=False))
    didx = np.sort(rng.choice(m, min(m, NSAMPLE), replace=False))
    eidx = np.sort(rng.choice(n, min(n, NSAMPLE), replace=False))
    unorm, vnorm, cgs, us, vs, kept, res_rows, times = [], [], [], [], [], [], [], []
    tl = [time.perf_counter()]

    def cb(state):
        unorm.append(np.linalg.norm(state.u))
        vnorm.append(np.linalg.norm(state.v))
        cgs.append(ws.cache.cg_iters_total)
        if state.iter in SNAP:
            us.append(state.u[idx].copy())
            vs.append(state.v[idx].copy())
            kept.append(state.iter)
        now = time.perf_counter()
        times.append(now - tl[0])
        tl[0] = now
        print(f"it {state.iter} {times[-1]:.2f}s |u|={unorm[-1]:.6e}", flush=True)

    orig = rsolver.check_termination

    def rec(state, data_, scal, settings, res=None):
        res_rows.append([float(getattr(res, f)) for f in RES_FIELDS])
        return orig(state, data_, scal, settings, res=res)

    rsolver.check_termination = rec
    try:
        t0 = time.perf_counter()
        sol = ws.solve(on_iteration=cb)
        solve_s = time.perf_counter() - t0
    finally:
        rsolver.check_termination = orig
    r = sol.info.residuals
    np.savez_compressed(
        out, cfg=json.dumps(CFG), m=m, n=n, nnz=rowidx.size, idx=idx, didx=didx, eidx=eidx,
        D=ws.scal.D[didx], E=ws.scal.E[eidx], sigma=ws.scal.sigma, rho=ws.scal.rho,
        g_sample=ws.cache.g[eidx] if getattr(ws.cache, "g", None) is not None else np.zeros(0),
        unorm=np.array(unorm), vnorm=np.array(vnorm), cg_total=np.array(cgs), kept=np.array(kept),
        us=np.array(us), vs=np.array(vs), res=np.array(res_rows),
        final_res=np.array([float(getattr(r, f)) for f in RES_FIELDS]),
        status=sol.status.value, iterations=sol.info.iterations, cg_iters=sol.info.cg_iters,
        settings=json.dumps(dict(max_iters=iters, eps=1e-3)), iter_seconds=np.array(times),
        setup_seconds=setup_s, solve_seconds=solve_s)
    print(f"status={sol.status.value} iters={sol.info.iterations} cg={sol.info.cg_iters} "
          f"solve {solve_s:.1f}s -> {out}", flush=True)


if __name__ == "__main__":
    main()
