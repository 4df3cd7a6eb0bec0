"""Setup-time breakdown (SCS_DEBUG timestamps) for the bench's time-to-eps
shape at config 5 size: python tools/r02_setup_probe.py [c5|c3]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SCS_DEBUG"] = "1"
import bench  # noqa: E402
import paper_1312_3039_b200 as P  # noqa: E402

cfg = bench.TTE[sys.argv[1] if len(sys.argv) > 1 else "c5"]
colptr, rowidx, vals, b, c, cone = bench.load_problem(cfg)
A = object.__new__(P.SparseMatrix)
A.nrows, A.ncols, A.colptr, A.rowidx, A.vals = b.size, colptr.size - 1, colptr, rowidx, vals
data = object.__new__(P.ProblemData)
data.A, data.b, data.c, data.spec = A, b, c, P.ConeSpec.from_any(cone)
for rep in range(2):  # the second one: CUDA context and module loads already paid
    t0 = time.perf_counter()
    ws = P.Workspace(data, P.Settings(max_iters=10))
    print(f"setup {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
    del ws
