"""Find where a config-4 solve goes non-finite (debug)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1312_3039_b200 as P
from paper_1312_3039_b200 import generators as G, native

p = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
lam = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
prob = G.gen_portfolio_c4(p, 10, p // 10, seed=1, lam=lam, kappa=lam)
colptr, ri, va, b, c, cone = prob
m, n = b.size, colptr.size - 1
data = P.ProblemData(P.SparseMatrix(m, n, colptr, ri, va), b, c, P.ConeSpec.from_any(cone))
ws = P.Workspace(data, P.Settings(max_iters=50000))
last = {}
def cb(s):
    if True:
        if 'u' in last:
            last['pu'], last['pv'] = last['u'], last['v']
        last['u'], last['v'], last['k'] = s.u.copy(), s.v.copy(), s.iter
        bad = ~np.isfinite(s.u) | ~np.isfinite(s.v)
        mx = np.abs(s.u).max()
        if s.iter % 500 == 0:
            print(s.iter, 'max|u|', mx, 'max|v|', np.abs(s.v).max(), 'tau', s.u[-1], 'kappa', s.v[-1], flush=True)
        if bad.any():
            idx = np.flatnonzero(bad)
            print('nonfinite at', s.iter, idx[:10], 'count', idx.size, 'n', n, 'bounds', n + cone['z'] + cone['l'], n + cone['z'] + cone['l'] + sum(cone['q']), flush=True)
            np.savez('gpurun_out/c4_nan_state.npz', u=last.get('pu'), v=last.get('pv'), u_bad=s.u, v_bad=s.v, k=s.iter)
            raise SystemExit
try:
    sol = ws.solve(on_iteration=cb)
    print(sol.status, sol.info.iterations)
except Exception as e:
    print('EXC', e, 'last ok iter', last.get('k'))
    np.savez('gpurun_out/c4_nan_state.npz', u=last['u'], v=last['v'], k=last['k'])
    u, v = last['u'], last['v']
    z, l = cone['z'], cone['l']
    off = n + z + l + sum(cone['q']) + sum(k * (k + 1) // 2 for k in cone['s'])
    ue, ve = u[off:off + 3 * cone['ep']].reshape(-1, 3), v[off:off + 3 * cone['ep']].reshape(-1, 3)
    print('exp u range', ue.min(0), ue.max(0), 'v range', ve.min(0), ve.max(0))
    print('max|u| per part: x', np.abs(u[:n]).max(), 'y', np.abs(u[n:-1]).max(), 'tau', u[-1], v[-1])
