"""Generate golden fixtures by running the REFERENCE (conesplit 0.1.0).

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed):
  known_answers.json   SPEC.md / test_cones.py known-answer values
  cones.npz            random inputs and the reference's cone projections
  traj_<name>.npz      problem data, settings, the first <=50 (u, v) iterates
                       from Workspace.solve(on_iteration=...) and the final
                       Solution of the reference's indirect solver
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
from conesplit import embedding as remb  # noqa: E402
from conesplit import sparse_linalg as rsl  # noqa: E402

from paper_1312_3039_b200 import generators as gen  # noqa: E402

N_TRAJ = 50


def to_ref(colptr, rowidx, vals, b, c, cone, m=None, n=None):
    n = colptr.size - 1 if n is None else n
    m = b.size if m is None else m
    A = rsl.SparseMatrix(m, n, colptr, rowidx, vals)
    spec = rcones.ConeSpec(zero_dim=cone.get("z", 0), nonneg_dim=cone.get("l", 0),
                           soc_dims=tuple(cone.get("q", ())),
                           psd_sides=tuple(cone.get("s", ())))
    return ref.ProblemData(A, b, c, spec)


def from_ref(data):
    sp = data.spec
    return (data.A.colptr, data.A.rowidx, data.A.vals, data.b, data.c,
            {"z": sp.zero_dim, "l": sp.nonneg_dim, "q": list(sp.soc_dims),
             "s": list(sp.psd_sides), "ep": 0})


def dump_traj(name, data, settings, snapshots=None, nsample=4000):
    """Every iterate k <= 50 is kept: in full (snapshots=None), or -- for
    the big config-2 problems -- as a seeded sample of `nsample` entries of
    (u, v) at every k plus the full vectors at the `snapshots`.  The norms
    ||u||, ||v|| and the cumulative CG count are kept for every k <= 50."""
    us, vs, kept, unorm, vnorm, cgs, su, sv = [], [], [], [], [], [], [], []
    ell = data.n + data.m + 1
    sidx = np.sort(np.random.default_rng(99).choice(ell, min(ell, nsample), replace=False))
    box = {}

    def cb(state):
        k = state.iter
        if k > N_TRAJ:
            return
        unorm.append(np.linalg.norm(state.u))
        vnorm.append(np.linalg.norm(state.v))
        cgs.append(box["ws"].cache.cg_iters_total)
        if snapshots is not None:
            su.append(state.u[sidx].copy())
            sv.append(state.v[sidx].copy())
        if snapshots is None or k in snapshots:
            us.append(state.u.copy())
            vs.append(state.v.copy())
            kept.append(k)

    t0 = time.perf_counter()
    ws = ref.Workspace(data, settings)
    box["ws"] = ws
    sol = ws.solve(on_iteration=cb)
    dt = time.perf_counter() - t0
    colptr, rowidx, vals, b, c, cone = from_ref(data)
    res = sol.info.residuals
    out = dict(
        m=data.m, n=data.n, colptr=colptr, rowidx=rowidx.astype(np.int32), vals=vals,
        b=b, c=c, cone=json.dumps(cone),
        settings=json.dumps({k: getattr(settings, k) for k in (
            "alpha", "max_iters", "eps_pri", "eps_dual", "eps_gap", "eps_infeas",
            "eps_unbdd", "check_interval", "cg_max", "cg_tol", "normalize", "sweeps")}),
        us=np.array(us), vs=np.array(vs), kept=np.array(kept, np.int64),
        unorm=np.array(unorm), vnorm=np.array(vnorm), cg_total=np.array(cgs, np.int64),
        status=sol.status.value, iterations=sol.info.iterations,
        cg_iters=sol.info.cg_iters,
        primal_obj=sol.primal_obj, dual_obj=sol.dual_obj,
        pri_res=sol.info.pri_res, dual_res=sol.info.dual_res, gap=sol.info.gap,
        u_final=ws.final_state.u, v_final=ws.final_state.v,
        D=ws.scal.D, E=ws.scal.E, sigma=ws.scal.sigma, rho=ws.scal.rho,
        g=ws.cache.g, denom=ws.cache.denom,
        res=np.array([res.pri_norm, res.dual_norm, res.gap, res.pri_thresh,
                      res.dual_thresh, res.gap_thresh, res.unbdd_measure,
                      res.infeas_measure]),
        ref_seconds=dt,
    )
    if snapshots is not None:
        out.update(sidx=sidx, us_sample=np.array(su), vs_sample=np.array(sv))
    for key in ("x", "y", "s", "certificate", "certificate_unbounded"):
        val = getattr(sol, key)
        if val is not None:
            out[key] = val
    np.savez_compressed(os.path.join(HERE, f"traj_{name}.npz"), **out)
    print(f"{name:22s} m={data.m:6d} n={data.n:6d} nnz={data.A.nnz:7d} "
          f"{sol.status.value:18s} it={sol.info.iterations:5d} "
          f"cg={sol.info.cg_iters:6d} {dt:6.2f}s")


def known_answers():
    SM = rsl.SparseMatrix
    ka = {}
    A = SM.from_dense([[1.0, 0.0], [0.0, 2.0]])
    ka["spmv"] = rsl.spmv(A, np.array([3.0, 4.0])).tolist()
    ka["spmv_empty"] = rsl.spmv(SM(2, 3, np.zeros(4, np.int64), [], []),
                                np.ones(3)).tolist()
    d = ref.ProblemData(SM.from_dense([[1.0]]), np.array([1.0]), np.array([1.0]),
                        rcones.ConeSpec(nonneg_dim=1))
    ka["apply_q"] = remb.apply_q(d, np.array([1.0, 0.0, 0.0])).tolist()
    cache = remb.setup_cache(d, mode="indirect")
    ka["setup_g"] = cache.g.tolist()
    ka["setup_denom"] = float(cache.denom)
    cache2 = remb.setup_cache(d, mode="indirect")
    ka["solve_kkt"] = remb.solve_kkt(cache2, d, np.array([1.0, 1.0])).tolist()  # :239
    cache3 = remb.setup_cache(d, mode="indirect")
    ka["project_affine"] = remb.project_affine(cache3, d, np.array([1.0, 1.0, 1.0])).tolist()
    ka["soc_boundary"] = rcones.project_primal_cone(
        [0.0, 3.0, 4.0], rcones.ConeSpec(soc_dims=(3,))).tolist()      # test_cones.py:88-94
    ka["soc_polar"] = rcones.project_primal_cone(
        [-5.0, 3.0, 4.0], rcones.ConeSpec(soc_dims=(3,))).tolist()
    ka["embedding_basic"] = rcones.project_embedding_cone(
        [-2.0, -1.0, -3.0], 1, rcones.ConeSpec(nonneg_dim=1)).tolist()  # :145-149
    ka["embedding_zero"] = rcones.project_embedding_cone(
        [7.0, -1.0], 0, rcones.ConeSpec(zero_dim=1)).tolist()           # :157-160
    x = rcones.pack_symmetric(np.diag([1.0, -1.0]))
    ka["psd_diag_in"] = x.tolist()
    ka["psd_diag_out"] = rcones.project_primal_cone(
        x, rcones.ConeSpec(psd_sides=(2,))).tolist()                    # :105-109
    with open(os.path.join(HERE, "known_answers.json"), "w") as fh:
        json.dump(ka, fh, indent=1)


def cone_fixture():
    rng = np.random.default_rng(1234)
    specs = [
        dict(z=2, l=3, q=[3, 4], s=[2, 3]),      # test_cones.py:20 MIXED_SPEC
        dict(z=0, l=5, q=[1, 2, 7, 33], s=[1, 4, 6, 8]),
        dict(z=3, l=0, q=[100], s=[10, 16]),
    ]
    out = {"specs": json.dumps(specs)}
    for i, sp in enumerate(specs):
        spec = rcones.ConeSpec(sp["z"], sp["l"], tuple(sp["q"]), tuple(sp["s"]))
        X = 2.0 * rng.standard_normal((20, spec.total_dim))
        out[f"x{i}"] = X
        out[f"dual{i}"] = np.array([rcones.project_dual_cone(x, spec) for x in X])
        out[f"primal{i}"] = np.array([rcones.project_primal_cone(x, spec) for x in X])
    np.savez_compressed(os.path.join(HERE, "cones.npz"), **out)


def main():
    known_answers()
    cone_fixture()
    S = ref.Settings
    SM = rsl.SparseMatrix
    tiny_lp = ref.ProblemData(SM.from_dense([[-1.0]]), np.array([-1.0]),
                              np.array([1.0]), rcones.ConeSpec(nonneg_dim=1))
    tiny_inf = ref.ProblemData(SM.from_dense([[1.0], [-1.0]]), np.array([0.0, -1.0]),
                               np.array([0.0]), rcones.ConeSpec(nonneg_dim=2))
    tiny_unb = ref.ProblemData(SM.from_dense([[-1.0]]), np.array([0.0]),
                               np.array([-1.0]), rcones.ConeSpec(nonneg_dim=1))
    ind = dict(linsys_mode="indirect")
    dump_traj("tiny_lp", tiny_lp, S(**ind))
    dump_traj("tiny_infeasible", tiny_inf, S(**ind))
    dump_traj("tiny_unbounded", tiny_unb, S(**ind))
    for kind in ("lp_feasible", "lp_infeasible", "lp_unbounded"):
        dump_traj(f"ref_{kind}", ref.generators.gen_lp_family(kind, 20, 40, 3),
                  S(**ind))
    dump_traj("ref_lasso", ref.generators.gen_lasso(30, 12, 1), S(**ind))
    dump_traj("ref_portfolio", ref.generators.gen_portfolio(40, 5, 1), S(**ind))
    dump_traj("ref_rpca", ref.generators.gen_rpca(4, 1, 1), S(**ind, max_iters=400))
    mix = gen.gen_planted(dict(z=4, l=30, q=[5, 5, 9], s=[2, 3, 4, 5]), 25, 0.25, 7)
    dump_traj("mixed", to_ref(*mix), S(**ind, eps_pri=1e-5, eps_dual=1e-5,
                                       eps_gap=1e-5))
    dump_traj("mixed_ci3_cg5", to_ref(*mix), S(**ind, check_interval=3, cg_max=5,
                                               alpha=1.2))
    dump_traj("mixed_nonorm_cgtol", to_ref(*mix), S(**ind, normalize=False,
                                                    cg_tol=1e-7))
    # config 1: LP+SOC m=3000 n=1000 1% dense, eps=1e-5 (BASELINE.json configs[0])
    c1 = gen.gen_lp_soc(3000, 1000, 0.01, 100, 10, seed=0)
    eps5 = dict(eps_pri=1e-5, eps_dual=1e-5, eps_gap=1e-5, eps_infeas=1e-5,
                eps_unbdd=1e-5)
    dump_traj("c1_lp_soc", to_ref(*c1), S(**ind, **eps5, max_iters=5000))
    # config 2: infeasible / unbounded m=30000 n=10000 (BASELINE.json configs[1])
    for kind in ("lp_infeasible", "lp_unbounded"):
        c2 = gen.gen_lp(kind, 10000, 30000, seed=2)
        dump_traj(f"c2_{kind}", to_ref(*c2), S(**ind, **eps5), snapshots=(1, 2, 10, 50))
    # the post-loop status rule (solver.py:364-369): MAX_ITERS_REACHED when
    # tau > 1e-8 ||u|| at max_iters, else INDETERMINATE.  The LASSO shape
    # q = 18 p is the BASELINE regime where the reference stalls.
    dump_traj("maxit_lasso_q18p", ref.generators.gen_lasso(10, 180, 1), S(**ind, max_iters=400))
    lpi = ref.generators.gen_lp_family("lp_infeasible", 20, 40, 3)
    never = dict(eps_infeas=1e-300, eps_unbdd=1e-300)  # certificates never accepted
    dump_traj("maxit_lp_infeasible", lpi, S(**ind, **never, max_iters=10))
    dump_traj("indet_lp_infeasible", lpi, S(**ind, **never, max_iters=100))


if __name__ == "__main__":
    main()
