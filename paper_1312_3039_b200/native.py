"""ctypes binding of the C-ABI in include/scs_b200.h.

The library is built in-tree (``python -m paper_1312_3039_b200.build`` or
``__graft_entry__.build()``) as ``paper_1312_3039_b200/libscs_b200.so``.
There is no fallback: every solver entry point raises if the library is
missing or fails to load.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libscs_b200.so")

SCS_OK = 0
ERRORS = {
    -1: "EINVAL", -2: "ENONFINITE", -3: "ESETUP", -4: "ENOCONV",
    -5: "ECUDA", -6: "ENCCL", -7: "ENOMEM",
}

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)

# every exported symbol of include/scs_b200.h
EXPORTS = (
    "scs_create", "scs_solve", "scs_begin", "scs_step", "scs_finish",
    "scs_get_state", "scs_get_scaling", "scs_update_vectors",
    "scs_point_residuals", "scs_extract_point", "scs_apply_a", "scs_project_cone", "scs_destroy",
    "scs_last_error", "scs_abi_version", "scs_nccl_unique_id",
    "scs_partition_rows", "scs_gen_lasso", "scs_bench_iters", "scs_bench_kernel", "scs_query",
    "scs_host_alloc", "scs_host_free",
    "scs_emu_group_create", "scs_emu_group_destroy", "scs_allreduce",
    "scs_cone_margin_count", "scs_cone_margins", "scs_check_products",
)


class Problem(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("colptr", i64p), ("rowidx", i64p),
                ("vals", f64p), ("b", f64p), ("c", f64p), ("z", C.c_int64), ("l", C.c_int64),
                ("nq", C.c_int64), ("q", i64p), ("ns", C.c_int64), ("s", i64p),
                ("ep", C.c_int64), ("m_global", C.c_int64), ("row_lo", C.c_int64)]


class SettingsC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("max_iters", C.c_int64), ("eps_pri", C.c_double),
                ("eps_dual", C.c_double), ("eps_gap", C.c_double), ("eps_infeas", C.c_double),
                ("eps_unbdd", C.c_double), ("check_interval", C.c_int64), ("cg_max", C.c_int64),
                ("cg_tol", C.c_double), ("normalize", C.c_int32), ("sweeps", C.c_int32),
                ("device", C.c_int32), ("fast", C.c_int32)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.POINTER(C.c_uint8)),
                ("emu_group", C.c_void_p), ("bounds", C.POINTER(C.c_int64)),
                ("flags", C.c_int32), ("pad_", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("status", C.c_int32), ("pad_", C.c_int32), ("iterations", C.c_int64),
                ("cg_iters", C.c_int64), ("res", C.c_double * 8), ("setup_seconds", C.c_double),
                ("solve_seconds", C.c_double), ("launches", C.c_int64)]


_lib = None


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


def load():
    """Load (once) and type the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"native library {LIB_PATH} is missing: run `python -m paper_1312_3039_b200.build`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    hp = C.c_void_p
    sig = {
        "scs_create": (C.c_int, [C.POINTER(Problem), C.POINTER(SettingsC), C.POINTER(Dist),
                                 C.POINTER(hp)]),
        "scs_solve": (C.c_int, [hp, f64p, f64p, f64p, C.POINTER(Info)]),
        "scs_begin": (C.c_int, [hp, f64p, f64p, f64p]),
        "scs_step": (C.c_int, [hp, C.c_int64, C.POINTER(Info)]),
        "scs_finish": (C.c_int, [hp, C.POINTER(Info)]),
        "scs_get_state": (C.c_int, [hp, f64p, f64p]),
        "scs_get_scaling": (C.c_int, [hp, f64p, f64p, f64p, f64p]),
        "scs_update_vectors": (C.c_int, [hp, f64p, f64p]),
        "scs_point_residuals": (C.c_int, [hp, f64p, f64p, f64p, f64p]),
        "scs_extract_point": (C.c_int, [hp, f64p, f64p, f64p, f64p]),
        "scs_apply_a": (C.c_int, [hp, C.c_int, f64p, f64p]),
        "scs_project_cone": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, i64p, C.c_int64, i64p,
                                       C.c_int64, C.c_int, C.c_int64, f64p, f64p, C.c_int]),
        "scs_bench_iters": (C.c_int, [hp, C.c_int64, f64p]),
        "scs_cone_margin_count": (C.c_int64, [C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int64, C.c_int32]),
        "scs_check_products": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, f64p, f64p, f64p,
                                         f64p, f64p, C.c_int32]),
        "scs_cone_margins": (C.c_int, [f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, i64p,
                                       C.c_int64, i64p, C.c_int64, C.c_int32, C.c_int32, f64p,
                                       C.c_int64]),
        "scs_bench_kernel": (C.c_int, [hp, C.c_int, C.c_int64, f64p, f64p]),
        "scs_query": (C.c_int, [hp, C.c_int32, i64p]),
        "scs_host_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
        "scs_host_free": (None, [C.c_void_p]),
        "scs_destroy": (None, [hp]),
        "scs_emu_group_create": (C.c_void_p, [C.c_int32]),
        "scs_emu_group_destroy": (None, [C.c_void_p]),
        "scs_allreduce": (C.c_int, [hp, f64p, C.c_int64]),
        "scs_last_error": (C.c_char_p, [hp]),
        "scs_abi_version": (C.c_int, []),
        "scs_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "scs_partition_rows": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, i64p, C.c_int64, i64p,
                                         C.c_int64, i64p, C.c_int32, i64p]),
        "scs_gen_lasso": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64,
                                    C.c_int64, C.c_int, i64p, i64p, i64p, i64p, i64p, f64p,
                                    f64p, f64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a, typ=f64p):
    if a is None:
        return C.cast(None, typ)
    return a.ctypes.data_as(typ)


def check(rc, handle=None):
    if rc != SCS_OK:
        lib = load()
        msg = lib.scs_last_error(handle).decode(errors="replace")
        raise NativeError(rc, msg)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def project_cone(x, cone, kind="dual", n=0, device=0):
    """Device cone projection (scs_project_cone): kind dual | primal | embedding."""
    lib = load()
    x = f64(x)
    out = np.empty_like(x)
    q = i64(cone.get("q", ()))
    s = i64(cone.get("s", ()))
    k = {"dual": 0, "primal": 1, "embedding": 2}[kind]
    check(lib.scs_project_cone(int(cone.get("z", 0)), int(cone.get("l", 0)), q.size,
                               ptr(q, i64p), s.size, ptr(s, i64p), int(cone.get("ep", 0)),
                               k, int(n), ptr(x), ptr(out), int(device)))
    return out


def cone_margins(vec, cone, dual=False, device=0):
    """Device cone-membership margins per block (scs_cone_margins)."""
    lib = load()
    vec = f64(vec)
    q = i64(cone.get("q", ()))
    s = i64(cone.get("s", ()))
    z, l, ep = int(cone.get("z", 0)), int(cone.get("l", 0)), int(cone.get("ep", 0))
    cnt = lib.scs_cone_margin_count(z, l, q.size, s.size, ep, int(bool(dual)))
    out = np.empty(cnt, np.float64)
    check(lib.scs_cone_margins(ptr(vec), vec.size, z, l, q.size, ptr(q, i64p), s.size,
                               ptr(s, i64p), ep, int(bool(dual)), int(device), ptr(out), cnt))
    return out


def check_products(A, x=None, y=None, device=0):
    """Device A x and/or A^T y of a CSC SparseMatrix (scs_check_products)."""
    lib = load()
    cp, ri, va = i64(A.colptr), i64(A.rowidx), f64(A.vals)
    ax = np.empty(A.nrows) if x is not None else None
    aty = np.empty(A.ncols) if y is not None else None
    xx = f64(x) if x is not None else None
    yy = f64(y) if y is not None else None
    check(lib.scs_check_products(A.nrows, A.ncols, ptr(cp, i64p), ptr(ri, i64p), ptr(va),
                                 ptr(xx), ptr(yy), ptr(ax), ptr(aty), int(device)))
    return ax, aty


class _PinnedPool:
    """Page-locked float64 buffers (scs_host_alloc), recycled: a buffer goes
    back to the pool when the last numpy array viewing it is collected, so
    repeated solves of one size reuse the same pinned pages."""

    def __init__(self):
        self._free = {}
        self._lock = threading.Lock()

    def empty(self, count):
        count = int(count)
        if count <= 0:
            return np.empty(0)
        nbytes = 8 * count
        with self._lock:
            lst = self._free.get(nbytes)
            ptr = lst.pop() if lst else None
        if ptr is None:
            p = C.c_void_p()
            check(load().scs_host_alloc(nbytes, C.byref(p)))
            ptr = p.value
        buf = (C.c_double * count).from_address(ptr)
        weakref.finalize(buf, self._release, nbytes, ptr)
        return np.frombuffer(buf, dtype=np.float64, count=count)

    def _release(self, nbytes, ptr):
        with self._lock:
            self._free.setdefault(nbytes, []).append(ptr)


_pool = _PinnedPool()


def pinned_empty(count):
    """Uninitialised page-locked float64 vector of length `count`."""
    return _pool.empty(count)


def pinned_zeros(count):
    a = _pool.empty(count)
    a[:] = 0.0
    return a


(Q_FORMAT_A, Q_FORMAT_AT, Q_LAUNCHES_PER_ITER, Q_STREAM_BYTES_A, Q_STREAM_BYTES_AT,
 Q_CG_ITERS_TOTAL) = range(6)


def query(h, key):
    """scs_query: layout facts of a handle (SpMV format per matrix, ...)."""
    out = C.c_int64()
    check(load().scs_query(h, int(key), C.byref(out)), h)
    return int(out.value)


def gen_lasso(p, q, nnz_f, seed=1, row_lo=0, row_hi=0, threads=0):
    """Huge sparse-F LASSO (C generator) -> (colptr, rowidx, vals, b, c, cone)."""
    lib = load()
    m, n, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib.scs_gen_lasso(p, q, nnz_f, seed, row_lo, row_hi, threads, C.byref(m), C.byref(n),
                            C.byref(nnz), None, None, None, None, None))
    colptr = np.empty(n.value + 1, np.int64)
    rowidx = np.empty(nnz.value, np.int64)
    vals = np.empty(nnz.value, np.float64)
    b = np.empty(m.value, np.float64)
    c = np.empty(n.value, np.float64)
    check(lib.scs_gen_lasso(p, q, nnz_f, seed, row_lo, row_hi, threads, C.byref(m), C.byref(n),
                            C.byref(nnz), ptr(colptr, i64p), ptr(rowidx, i64p), ptr(vals),
                            ptr(b), ptr(c)))
    cone = {"z": 0, "l": 2 * p, "q": [q + 2], "s": [], "ep": 0}
    return colptr, rowidx, vals, b, c, cone


def partition_rows(cone, row_nnz, world):
    lib = load()
    q = i64(cone.get("q", ()))
    s = i64(cone.get("s", ()))
    rn = i64(row_nnz)
    out = np.empty(world + 1, np.int64)
    check(lib.scs_partition_rows(int(cone.get("z", 0)), int(cone.get("l", 0)), q.size,
                                 ptr(q, i64p), s.size, ptr(s, i64p), int(cone.get("ep", 0)),
                                 ptr(rn, i64p), int(world), ptr(out, i64p)))
    return out
