"""Row sharding of the hot path over several GPUs.

Rank k owns rows [bounds[k], bounds[k+1]) of A (its CSR(A_k) and
CSR(A_k^T)), the matching slices of every m-length vector, and a replica of
every n-length vector; the CG of the subspace projection runs replicated.
The exchange steps are NCCL all-reduces of the A^T-pass partial products
and of the y-part scalars (plus the partial norms of second-order cones
that straddle a bound).  Bounds come from ``scs_partition_rows``: never
inside a PSD or exponential block, balanced by nonzeros.

Ranks are one process per GPU joined by NCCL (``nccl_bootstrap`` uses
torch.distributed only to broadcast the 128-byte NCCL id), or -- to test the
sharded path with a single GPU -- one host thread per shard joined by an
in-process emulated group (``emulated_solve``), or one process per shard
joined by a host shared-memory group (``host_bootstrap``).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from . import native


@dataclass
class ShardSpec:
    rank: int
    world: int
    bounds: np.ndarray
    nccl_id: bytes = None
    emu_group: int = None     # scs_emu_group* (emulated group)
    force: bool = False       # sharded code path even with world == 1
    host_name: str = None     # POSIX shared-memory group name (one process per shard, one node)


class ShardProblem:
    """Rows [row_lo, row_lo + m) of a global problem: CSC of that row slice
    (local row indices), b of the slice, the full c and the global cone."""

    def __init__(self, colptr, rowidx, vals, b, c, spec, row_lo, m_global):
        from .api import ConeSpec

        self.colptr = native.i64(colptr)
        self.rowidx = native.i64(rowidx)
        self.vals = native.f64(vals)
        self.b = native.f64(b)
        self.c = native.f64(c)
        self.spec = ConeSpec.from_any(spec)
        self.row_lo = int(row_lo)
        self.m_global = int(m_global)
        if self.spec.total_dim != self.m_global:
            raise ValueError("cone dimension does not match the global row count")

    @property
    def m(self):
        return self.b.size

    @property
    def n(self):
        return self.c.size


def row_bounds(cone, rowidx, m, world):
    """Shard bounds balancing nonzeros, never cutting PSD/exp blocks."""
    row_nnz = np.bincount(np.asarray(rowidx, np.int64), minlength=m)
    return native.partition_rows(cone, row_nnz, world)


def slice_rows(colptr, rowidx, vals, lo, hi):
    """CSC of rows [lo, hi) with local row indices."""
    colptr = np.asarray(colptr, np.int64)
    rowidx = np.asarray(rowidx, np.int64)
    n = colptr.size - 1
    keep = (rowidx >= lo) & (rowidx < hi)
    cols = np.repeat(np.arange(n), np.diff(colptr))[keep]
    cp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=cp[1:])
    return cp, rowidx[keep] - lo, np.asarray(vals, np.float64)[keep]


def shard_problem(colptr, rowidx, vals, b, c, cone, bounds, rank):
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    cp, ri, va = slice_rows(colptr, rowidx, vals, lo, hi)
    return ShardProblem(cp, ri, va, np.asarray(b)[lo:hi], c, cone, lo, int(bounds[-1]))


def emulated_solve(prob, settings, world, bounds=None, warm_start=None, on_iteration=None):
    """Solve one problem as `world` row shards on one GPU (threads + an
    emulated all-reduce group).  Returns [(Workspace, Solution)] per rank."""
    from .api import Workspace

    colptr, rowidx, vals, b, c, cone = prob
    m = np.asarray(b).size
    if bounds is None:
        bounds = row_bounds(cone, rowidx, m, world)
    lib = native.load()
    group = lib.scs_emu_group_create(world)
    out = [None] * world
    errs = [None] * world

    def run(rank):
        try:
            shard = shard_problem(colptr, rowidx, vals, b, c, cone, bounds, rank)
            spec = ShardSpec(rank, world, bounds, emu_group=group, force=True)
            ws = Workspace(shard, settings, dist=spec)
            ws_start = None
            if warm_start is not None:
                x0, y0, s0 = warm_start
                lo, hi = int(bounds[rank]), int(bounds[rank + 1])
                ws_start = (x0, np.asarray(y0)[lo:hi], np.asarray(s0)[lo:hi])
            cb = (lambda st, r=rank: on_iteration(r, st)) if on_iteration else None
            sol = ws.solve(warm_start=ws_start, on_iteration=cb)
            out[rank] = (ws, sol)
        except BaseException as exc:  # surfaced below
            errs[rank] = exc

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    lib.scs_emu_group_destroy(group)
    for e in errs:
        if e is not None:
            raise e
    return out


def gather_vector(parts):
    """Concatenate per-rank slices of an m-length vector."""
    return np.concatenate([np.asarray(p) for p in parts])


def host_bootstrap(rank, world):
    """Name of a POSIX shared-memory group from rank 0, broadcast with
    torch.distributed (the process group must already be initialised): the
    host all-reduce joins one process per shard on one node without NCCL
    (e.g. two ranks sharing one GPU)."""
    import os
    import uuid

    import torch.distributed as dist

    obj = [f"/scs_{os.getpid()}_{uuid.uuid4().hex[:12]}" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def nccl_bootstrap(rank, world):
    """NCCL id from rank 0, broadcast with torch.distributed (plumbing only;
    the process group must already be initialised, e.g. gloo)."""
    import torch.distributed as dist

    obj = [None]
    if rank == 0:
        buf = (native.C.c_uint8 * 128)()
        native.check(native.load().scs_nccl_unique_id(buf))
        obj[0] = bytes(buf)
    dist.broadcast_object_list(obj, src=0)
    return obj[0]
