"""Worker for tests/test_gpu_multiproc.py: one rank of a world-size-2 run of
the CUDA row-sharded path on one GPU -- gloo bootstrap, a host shared-memory
group for the all-reduces (NCCL refuses two ranks on one device), per-rank
generation of its own rows (scs_gen_lasso row slice), the C-ABI solve --
writing its iterates (x-part, its y rows, tau) for the parent to compare."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(rank, world, port, out):
    import torch.distributed as dist

    import paper_1312_3039_b200 as P
    from paper_1312_3039_b200 import native, parallel

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    p, q, nnzf = 300, 6000, 200_000
    full_m = 2 * p + q + 2
    w = np.empty(full_m, np.int64)
    w[:2 * p], w[2 * p:2 * p + 2], w[2 * p + 2:] = 2, 1, max(1, nnzf // q)
    cone = {"z": 0, "l": 2 * p, "q": [q + 2], "s": [], "ep": 0}
    bounds = native.partition_rows(cone, w, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    colptr, rowidx, vals, b, c, cone = native.gen_lasso(p, q, nnzf, seed=3, row_lo=lo, row_hi=hi)
    name = parallel.host_bootstrap(rank, world)
    shard = parallel.ShardProblem(colptr, rowidx, vals, b, c, cone, lo, full_m)
    spec = parallel.ShardSpec(rank, world, bounds, host_name=name, force=True)
    ws = P.Workspace(shard, P.Settings(max_iters=60, eps_pri=1e-5, eps_dual=1e-5, eps_gap=1e-5),
                     dist=spec)
    us = {}
    sol = ws.solve(on_iteration=lambda s: us.__setitem__(s.iter, s.u.copy()) if s.iter <= 50
                   else None)
    ks = sorted(us)
    np.savez(out, ks=np.array(ks), us=np.array([us[k] for k in ks]), lo=lo, hi=hi,
             status=sol.status.value, iterations=sol.info.iterations, x=sol.x,
             y=sol.y if sol.y is not None else np.zeros(0))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
