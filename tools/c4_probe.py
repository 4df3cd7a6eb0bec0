"""Config 4 probe: per-iteration device time and convergence of the
full-size portfolio + exp + PSD instance (generators.gen_portfolio_c4)."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1312_3039_b200 as P  # noqa: E402
from paper_1312_3039_b200 import generators as G, native  # noqa: E402


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    prof = "--profile" in sys.argv
    t = time.perf_counter()
    colptr, rowidx, vals, b, c, cone = G.gen_portfolio_c4(p, 10, p // 10, seed=1)
    print(f"gen {time.perf_counter() - t:.2f}s m={b.size} n={colptr.size - 1} nnz={rowidx.size} "
          f"psd={len(cone['s'])} exp={cone['ep']}", flush=True)
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    t = time.perf_counter()
    ws = P.Workspace(data, P.Settings(max_iters=iters))
    print(f"setup {time.perf_counter() - t:.2f}s", flush=True)
    lib = native.load()
    h = ws._h
    native.check(lib.scs_begin(h, None, None, None), h)
    ms = native.C.c_double()
    native.check(lib.scs_bench_iters(h, 5, native.C.byref(ms)), h)
    if prof:
        rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
        rt.cudaProfilerStart()
        native.check(lib.scs_bench_iters(h, 1, native.C.byref(ms)), h)
        rt.cudaDeviceSynchronize()
        rt.cudaProfilerStop()
        return
    native.check(lib.scs_bench_iters(h, 50, native.C.byref(ms)), h)
    print(f"device ms/iteration {ms.value / 50:.4f}", flush=True)
    t = time.perf_counter()
    sol = ws.solve()
    dt = time.perf_counter() - t
    i = sol.info
    print(f"solve {dt:.2f}s status={sol.status.value} iters={i.iterations} pri={i.pri_res:.3e} "
          f"dual={i.dual_res:.3e} gap={i.gap:.3e} obj={sol.objective:.6g}", flush=True)


if __name__ == "__main__":
    main()
