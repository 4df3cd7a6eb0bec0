import os, sys, threading
sys.path.insert(0, "tests")
import numpy as np
import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import native, parallel
from _fixtures import load

d = load(sys.argv[1]); world = int(sys.argv[2])
prob = (d["colptr"], d["rowidx"], d["vals"], d["b"], d["c"], d["cone"])
colptr, rowidx, vals, b, c, cone = prob
m = b.size; n = colptr.size - 1
bounds = parallel.row_bounds(cone, rowidx, m, world)
print("bounds", bounds)
lib = native.load()
g = lib.scs_emu_group_create(world)
out = [None] * world
rng = np.random.default_rng(0)
x = rng.standard_normal(n); y = rng.standard_normal(m)
def run(r):
    sh = parallel.shard_problem(colptr, rowidx, vals, b, c, cone, bounds, r)
    ws = P.Workspace(sh, P.Settings(normalize=False), dist=parallel.ShardSpec(r, world, bounds, emu_group=g, force=True))
    lo, hi = bounds[r], bounds[r + 1]
    ax = ws.apply_a(x)
    aty = ws.apply_a(y[lo:hi], transpose=True)
    out[r] = (ax, aty, ws.tiled if hasattr(ws, "tiled") else None)
ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]

A = np.zeros((m, n)); cols = np.repeat(np.arange(n), np.diff(colptr)); A[rowidx, cols] = vals
ax = np.concatenate([o[0] for o in out])
ref = A @ x
for r in range(world):
    lo, hi = bounds[r], bounds[r+1]
    print("rank", r, "Ax err", np.abs(out[r][0] - ref[lo:hi]).max())
print("ATy err", [np.abs(o[1] - A.T @ y).max() for o in out])
if os.environ.get("SERIAL"):
    pass
