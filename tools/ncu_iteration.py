"""Profile one steady-state ADMM iteration of a bench config under ncu.

    ncu --profile-from-start off --set full ... python tools/ncu_iteration.py c5

Builds the bench workload, runs a few warm-up iterations, then brackets one
iteration (one graph launch) with cudaProfilerStart/Stop and, with --kernels,
one stand-alone launch of each roofline kernel (scs_bench_kernel).
"""

import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1312_3039_b200 as P  # noqa: E402
from paper_1312_3039_b200 import native  # noqa: E402


def cudart():
    for cand in ("/usr/local/cuda/lib64/libcudart.so", "libcudart.so", "libcudart.so.12"):
        try:
            return ctypes.CDLL(cand)
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    kernels = "--kernels" in sys.argv
    lib = native.load()
    colptr, rowidx, vals, b, c, cone = bench.load_problem(bench.CONFIGS[cfg_name])
    m, n = b.size, colptr.size - 1
    A = object.__new__(P.SparseMatrix)
    A.nrows, A.ncols, A.colptr, A.rowidx, A.vals = m, n, colptr, rowidx, vals
    data = object.__new__(P.ProblemData)
    data.A, data.b, data.c, data.spec = A, b, c, P.ConeSpec.from_any(cone)
    ws = P.Workspace(data, P.Settings(max_iters=100, eps_pri=1e-3, eps_dual=1e-3, eps_gap=1e-3))
    h = ws._h
    native.check(lib.scs_begin(h, None, None, None), h)
    ms = native.C.c_double()
    native.check(lib.scs_bench_iters(h, 4, native.C.byref(ms)), h)
    rt = cudart()
    rt.cudaProfilerStart()
    native.check(lib.scs_bench_iters(h, 1, native.C.byref(ms)), h)
    if kernels:
        kb = native.C.c_double()
        for kind in (0, 1):
            native.check(lib.scs_bench_kernel(h, kind, 1, native.C.byref(ms), native.C.byref(kb)), h)
    rt.cudaDeviceSynchronize()
    rt.cudaProfilerStop()
    print("done", cfg_name, m, n, flush=True)


if __name__ == "__main__":
    main()
