"""Worker for tests/test_multiproc_gloo.py: one rank of a world-size-2 gloo
group runs the row-sharded oracle and checks it against the unsharded one."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(rank, world, port, case, out):
    import torch
    import torch.distributed as dist

    from oracle import scs_oracle as O
    from oracle.sharded import ShardedOracle
    from paper_1312_3039_b200 import generators as G
    from paper_1312_3039_b200 import parallel

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).copy())
        dist.all_reduce(t)
        return t.numpy()

    if case == "mixed":
        prob = G.gen_planted(dict(z=4, l=30, q=[5, 5, 9], s=[2, 3], ep=2), 25, 0.25, 7)
        bounds = np.array([0, 36, prob[3].size], np.int64)  # cuts the first SOC
    else:
        prob = G.gen_lasso(40, 300, 3000, seed=2)
        bounds = parallel.row_bounds(prob[5], prob[1], prob[3].size, world)
    colptr, rowidx, vals, b, c, cone = prob
    m = b.size
    # unsharded reference trajectory (the pinned oracle)
    ref = O.OracleSolver(O.Csc(m, colptr.size - 1, colptr, rowidx, vals), b, c, cone,
                         max_iters=30)
    traj = {}
    ref.solve(on_iteration=lambda k, u, v: traj.__setitem__(k, u.copy()))
    sh = parallel.shard_problem(colptr, rowidx, vals, b, c, cone, bounds, rank)
    A = O.Csc(sh.m, sh.n, sh.colptr, sh.rowidx, sh.vals)
    so = ShardedOracle(A, sh.b, sh.c, cone, sh.row_lo, sh.m_global, allreduce)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    n = colptr.size - 1
    worst = 0.0
    for k, (ux, uy, ut) in enumerate(so.solve(30), start=1):
        u = traj[k]
        full = np.concatenate([u[:n], u[n + lo:n + hi], u[-1:]])
        mine = np.concatenate([ux, uy, [ut]])
        worst = max(worst, np.linalg.norm(mine - full) / max(np.linalg.norm(full), 1e-300))
    with open(out, "w") as fh:
        fh.write(repr(float(worst)))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5])
