import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G
for p in (300, 3000, 30000, 100000):
    for n_exp, ng, lam, kappa in ((p // 10, 0, 1.0, 1.0), (0, None, 1.0, 1.0),
                                  (p // 10, None, 1.0, 1.0), (p // 10, None, 0.1, 0.1),
                                  (p // 10, None, 10.0, 10.0)):
        prob = G.gen_portfolio_c4(p, 10, n_exp, n_groups=ng, seed=1, lam=lam, kappa=kappa)
        colptr, ri, va, b, c, cone = prob
        data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, ri, va), b, c,
                             P.ConeSpec.from_any(cone))
        t = time.time()
        sol = P.solve(data, P.Settings(max_iters=50000))
        print(p, n_exp, len(cone['s']), lam, kappa, sol.status.value, sol.info.iterations,
              round(time.time() - t, 2), sol.objective, flush=True)
