"""One steady-state ADMM iteration of BASELINE config 1 (LP+SOC 3000 x 1000)
under ncu: the per-kernel times of a launch-latency-bound iteration.

    ncu --profile-from-start off --metrics gpu__time_duration.sum ... python tools/ncu_c1.py
"""

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1312_3039_b200 as P  # noqa: E402
from paper_1312_3039_b200 import generators as G  # noqa: E402
from paper_1312_3039_b200 import native  # noqa: E402


def main():
    colptr, rowidx, vals, b, c, cone = G.gen_lp_soc(3000, 1000, 0.01, 100, 10, seed=0)
    data = P.ProblemData(P.SparseMatrix(b.size, colptr.size - 1, colptr, rowidx, vals), b, c,
                         P.ConeSpec.from_any(cone))
    ws = P.Workspace(data, P.Settings(max_iters=100, eps_pri=1e-9, eps_dual=1e-9, eps_gap=1e-9))
    lib, h = native.load(), ws._h
    native.check(lib.scs_begin(h, None, None, None), h)
    ms = native.C.c_double()
    native.check(lib.scs_bench_iters(h, 40, native.C.byref(ms)), h)  # past the first refresh
    rt = ctypes.CDLL("libcudart.so") if False else None
    for cand in ("/usr/local/cuda/lib64/libcudart.so", "libcudart.so", "libcudart.so.12"):
        try:
            rt = ctypes.CDLL(cand)
            break
        except OSError:
            continue
    rt.cudaProfilerStart()
    native.check(lib.scs_bench_iters(h, 1, native.C.byref(ms)), h)
    rt.cudaDeviceSynchronize()
    rt.cudaProfilerStop()
    native.check(lib.scs_bench_iters(h, 20, native.C.byref(ms)), h)
    print(f"c1 m={b.size} n={colptr.size - 1} nnz={rowidx.size} "
          f"{ms.value / 20 * 1e3:.1f} us/iteration (20 iterations, device)")


if __name__ == "__main__":
    main()
