import sys
sys.path.insert(0, "tests")
import numpy as np
import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import parallel
from _fixtures import load
d = load("ref_lp_infeasible")
colptr, rowidx, vals, b, c, cone = d["colptr"], d["rowidx"], d["vals"], d["b"], d["c"], d["cone"]
m = b.size; n = colptr.size - 1
for lo, hi in ((0, 21), (21, 40), (0, 40), (14, 27)):
    cp, ri, va = parallel.slice_rows(colptr, rowidx, vals, lo, hi)
    mk = hi - lo
    data = P.ProblemData(P.SparseMatrix(mk, n, cp, ri, va), b[lo:hi], c, P.ConeSpec(nonneg_dim=mk))
    ws = P.Workspace(data, P.Settings(normalize=False))
    A = np.zeros((mk, n)); cols = np.repeat(np.arange(n), np.diff(cp)); A[ri, cols] = va
    x = np.arange(n) + 1.0
    got = ws.apply_a(x)
    print(lo, hi, "nnz", va.size, "err", np.abs(got - A @ x).max())
    if np.abs(got - A @ x).max() > 1e-9:
        print(" rows bad:", np.nonzero(np.abs(got - A @ x) > 1e-9)[0])
        print(" row nnz:", np.bincount(ri, minlength=mk))
