"""Reference-facing Python surface (mirror of conesplit's public API).

Names, fields, argument meaning and error behaviour follow the reference
``conesplit`` 0.1.0 (/root/reference/pkg/src/conesplit):

* ``Settings`` (solver.py:52-84), ``Status`` (solver.py:43-49),
  ``SolveInfo`` (solver.py:96-105), ``Solution`` (solver.py:108-125),
  ``SolverState`` (solver.py:87-93), ``Residuals`` (scaling.py:37-55),
  ``ScalingData`` (scaling.py:18-34), ``SetupError`` (embedding.py:22-23);
* ``ConeSpec`` (cones.py:89-139) extended with ``exp_dim`` (3-dim
  exponential cones after the PSD blocks), ``SparseMatrix``
  (sparse_linalg.py:16-118, CSC), ``ProblemData`` (problem.py:15-53);
* ``Workspace`` (solver.py:291-378) and ``solve`` (solver.py:381-385), plus
  the north-star form ``solve(A, b, c, cone, settings)`` with the JSON cone
  dict ``{"z","l","q","s"[,"ep"]}`` (fileio.py:68-73);
* ``solution_to_dict`` (fileio.py:123-140).

Everything inside the iteration loop runs on the GPU through the C-ABI
(include/scs_b200.h).  The host keeps what the reference keeps outside the
loop: validation, settings checks and extract_solution's O(m+n) unscaling
(solver.py:251-288).  Only the indirect (CG) linear-system mode exists.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import native

TAU_EXTRACT_THRESHOLD = 1e-8  # solver.py:40


class SetupError(RuntimeError):
    """Raised when the linear-system cache cannot be constructed."""


class Status(Enum):
    SOLVED = "solved"
    INFEASIBLE = "infeasible"
    UNBOUNDED = "unbounded"
    INFEASIBLE_AND_UNBOUNDED = "infeasible_and_unbounded"
    INDETERMINATE = "indeterminate"
    MAX_ITERS_REACHED = "max_iters_reached"


_STATUS_BY_CODE = {0: Status.SOLVED, 1: Status.INFEASIBLE, 2: Status.UNBOUNDED,
                   3: Status.INFEASIBLE_AND_UNBOUNDED, 4: Status.INDETERMINATE,
                   5: Status.MAX_ITERS_REACHED}


@dataclass
class Settings:
    """Solver settings (solver.py:52-84).  linsys_mode must be "indirect":
    this framework replaces the reference's indirect (CG) path.  Opt-in
    modes, reported separately from parity mode:
    ``precond`` -- Jacobi-preconditioned CG on diag(I + A^T A) (changes the
    iterates); ``fast`` -- A x of the CG iterate by recurrence
    instead of a final matrix pass (rounding-level deviation)."""

    alpha: float = 1.5
    max_iters: int = 2500
    eps_pri: float = 1e-3
    eps_dual: float = 1e-3
    eps_gap: float = 1e-3
    eps_infeas: float = 1e-3
    eps_unbdd: float = 1e-3
    check_interval: int = 1
    linsys_mode: str = "indirect"
    cg_max: int = 2
    cg_tol: float = None
    normalize: bool = True
    sweeps: int = 10
    warm_start: tuple = None
    device: int = 0
    fast: bool = False
    precond: bool = False

    def __post_init__(self):
        if not 0.0 < self.alpha < 2.0:
            raise ValueError("alpha must lie in (0, 2)")
        for name in ("eps_pri", "eps_dual", "eps_gap", "eps_infeas", "eps_unbdd"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.max_iters < 1 or self.check_interval < 1:
            raise ValueError("max_iters and check_interval must be >= 1")
        if self.linsys_mode not in ("direct", "indirect"):
            raise ValueError("linsys_mode must be 'direct' or 'indirect'")
        if self.linsys_mode == "direct":
            raise ValueError("linsys_mode 'direct' (sparse LDL) is outside this framework's "
                             "scope; use 'indirect'")
        if self.cg_max < 1:
            raise ValueError("cg_max must be >= 1")
        if self.cg_tol is not None and not self.cg_tol > 0:
            raise ValueError("cg_solve: tol must be positive")
        if self.sweeps < 0:
            raise ValueError("sweeps must be >= 0")

    @classmethod
    def from_reference(cls, st, **over):
        """Convert a conesplit.Settings (forcing the indirect path)."""
        kw = {k: getattr(st, k) for k in (
            "alpha", "max_iters", "eps_pri", "eps_dual", "eps_gap", "eps_infeas", "eps_unbdd",
            "check_interval", "cg_max", "cg_tol", "normalize", "sweeps", "warm_start")}
        kw["linsys_mode"] = "indirect"
        kw.update(over)
        return cls(**kw)


@dataclass
class SolverState:
    u: np.ndarray
    v: np.ndarray
    iter: int = 0


@dataclass
class Residuals:
    pri_norm: float
    dual_norm: float
    gap: float
    pri_thresh: float
    dual_thresh: float
    gap_thresh: float
    unbdd_measure: float
    infeas_measure: float


@dataclass
class ScalingData:
    D: np.ndarray
    E: np.ndarray
    sigma: float
    rho: float


@dataclass
class SolveInfo:
    iterations: int = 0
    pri_res: float = np.nan
    dual_res: float = np.nan
    gap: float = np.nan
    setup_time: float = 0.0
    solve_time: float = 0.0
    cg_iters: int = 0
    residuals: Residuals = None


@dataclass
class Solution:
    status: Status
    x: np.ndarray = None
    y: np.ndarray = None
    s: np.ndarray = None
    certificate: np.ndarray = None
    certificate_unbounded: np.ndarray = None
    primal_obj: float = np.nan
    dual_obj: float = np.nan
    info: SolveInfo = field(default_factory=SolveInfo)

    @property
    def objective(self):
        """Average of primal and dual objectives (solver.py:122-125)."""
        return 0.5 * (self.primal_obj + self.dual_obj)


def packed_length(side):
    return side * (side + 1) // 2


@dataclass(frozen=True)
class ConeSpec:
    """Ordered cone blocks: zero, nonneg, SOC..., PSD..., exp x exp_dim."""

    zero_dim: int = 0
    nonneg_dim: int = 0
    soc_dims: tuple = field(default_factory=tuple)
    psd_sides: tuple = field(default_factory=tuple)
    exp_dim: int = 0

    def __post_init__(self):
        object.__setattr__(self, "soc_dims", tuple(int(d) for d in self.soc_dims))
        object.__setattr__(self, "psd_sides", tuple(int(s) for s in self.psd_sides))
        if self.zero_dim < 0 or self.nonneg_dim < 0 or self.exp_dim < 0:
            raise ValueError("cone dimensions must be nonnegative")
        if any(d < 1 for d in self.soc_dims):
            raise ValueError("second-order cone dims must be >= 1")
        if any(s < 1 for s in self.psd_sides):
            raise ValueError("PSD side lengths must be >= 1")

    @property
    def total_dim(self):
        return (self.zero_dim + self.nonneg_dim + sum(self.soc_dims)
                + sum(packed_length(s) for s in self.psd_sides) + 3 * self.exp_dim)

    def blocks(self):
        off = 0
        if self.zero_dim:
            yield ("zero", 0, self.zero_dim, 0)
            off += self.zero_dim
        if self.nonneg_dim:
            yield ("nonneg", off, self.nonneg_dim, 0)
            off += self.nonneg_dim
        for d in self.soc_dims:
            yield ("soc", off, d, 0)
            off += d
        for s in self.psd_sides:
            yield ("psd", off, packed_length(s), s)
            off += packed_length(s)
        for _ in range(self.exp_dim):
            yield ("exp", off, 3, 0)
            off += 3

    def to_dict(self):
        return {"z": self.zero_dim, "l": self.nonneg_dim, "q": list(self.soc_dims),
                "s": list(self.psd_sides), "ep": self.exp_dim}

    @classmethod
    def from_any(cls, cone):
        if isinstance(cone, ConeSpec):
            return cone
        if isinstance(cone, dict):
            return cls(int(cone.get("z", 0)), int(cone.get("l", 0)), tuple(cone.get("q", ())),
                       tuple(cone.get("s", ())), int(cone.get("ep", 0)))
        # reference conesplit.ConeSpec (duck-typed)
        return cls(int(cone.zero_dim), int(cone.nonneg_dim), tuple(cone.soc_dims),
                   tuple(cone.psd_sides), int(getattr(cone, "exp_dim", 0)))


@dataclass
class SparseMatrix:
    """CSC with int64 indices and float64 values (sparse_linalg.py:16-118)."""

    nrows: int
    ncols: int
    colptr: np.ndarray
    rowidx: np.ndarray
    vals: np.ndarray

    def __post_init__(self):
        self.colptr = np.ascontiguousarray(self.colptr, dtype=np.int64)
        self.rowidx = np.ascontiguousarray(self.rowidx, dtype=np.int64)
        self.vals = np.ascontiguousarray(self.vals, dtype=np.float64)
        self.validate()

    def validate(self):
        """sparse_linalg.py:34-54, same messages."""
        if self.nrows < 0 or self.ncols < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        if self.colptr.shape != (self.ncols + 1,):
            raise ValueError("colptr must have length ncols + 1")
        if self.colptr[0] != 0 or self.colptr[-1] != self.rowidx.size:
            raise ValueError("colptr must start at 0 and end at nnz")
        if np.any(np.diff(self.colptr) < 0):
            raise ValueError("colptr must be nondecreasing")
        if self.rowidx.size != self.vals.size:
            raise ValueError("rowidx and vals must have equal length")
        if self.rowidx.size:
            if self.rowidx.min() < 0 or self.rowidx.max() >= self.nrows:
                raise ValueError("row indices out of range")
            interior = np.ones(self.rowidx.size, dtype=bool)
            interior[self.colptr[:-1].clip(max=self.rowidx.size - 1)] = False
            if np.any(np.diff(self.rowidx)[interior[1:]] <= 0):
                raise ValueError("row indices must be strictly increasing per column")
        if not np.all(np.isfinite(self.vals)):
            raise ValueError("matrix values must be finite")

    @property
    def nnz(self):
        return self.vals.size

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @classmethod
    def from_dense(cls, mat):
        mat = np.asarray(mat, dtype=float)
        m, n = mat.shape
        cols, rows = np.nonzero(mat.T)
        colptr = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(cols, minlength=n), out=colptr[1:])
        return cls(m, n, colptr, rows, mat[rows, cols])

    @classmethod
    def from_any(cls, A):
        if isinstance(A, SparseMatrix):
            return A
        return cls(int(A.nrows), int(A.ncols), A.colptr, A.rowidx, A.vals)


@dataclass
class ProblemData:
    A: SparseMatrix
    b: np.ndarray
    c: np.ndarray
    spec: ConeSpec

    def __post_init__(self):
        self.b = np.ascontiguousarray(self.b, dtype=np.float64)
        self.c = np.ascontiguousarray(self.c, dtype=np.float64)
        validate_problem(self)

    @property
    def m(self):
        return self.A.nrows

    @property
    def n(self):
        return self.A.ncols


def validate_problem(data):
    """problem.py:38-53 (same checks, same messages)."""
    data.A.validate()
    m, n = data.A.nrows, data.A.ncols
    if data.b.shape != (m,):
        raise ValueError(f"b has shape {data.b.shape}, expected ({m},)")
    if data.c.shape != (n,):
        raise ValueError(f"c has shape {data.c.shape}, expected ({n},)")
    if not np.all(np.isfinite(data.b)):
        raise ValueError("b must be finite")
    if not np.all(np.isfinite(data.c)):
        raise ValueError("c must be finite")
    if data.spec.total_dim != m:
        raise ValueError(f"cone dimension {data.spec.total_dim} does not match row count {m}")


def as_problem(data) -> ProblemData:
    """Accept our ProblemData or the reference's (duck-typed)."""
    if isinstance(data, ProblemData):
        return data
    return ProblemData(SparseMatrix.from_any(data.A), data.b, data.c,
                       ConeSpec.from_any(data.spec))


def _raise(exc: native.NativeError, setup=False):
    if exc.code == -3:
        raise SetupError(exc.msg) from None
    if exc.code in (-1, -2):
        raise (SetupError if setup else ValueError)(exc.msg) from None
    raise RuntimeError(exc.msg) from None


class _CacheView:
    """The one EmbeddingCache field a caller reads (embedding.py:43)."""

    def __init__(self, cg_iters_total):
        self.cg_iters_total = cg_iters_total


class Workspace:
    """Reusable device-resident solver handle (solver.py:291-378).

    Setup (device transpose, equilibration, g = M^-1 h) happens once in the
    constructor; solves reuse it; update_vectors swaps b and/or c.
    ``dist`` = (rank, world, nccl_id bytes) for row-sharded runs, in which
    case ``data`` holds this rank's row slice (see parallel.shard_problem).
    """

    def __init__(self, data, settings=None, dist=None):
        self.settings = settings if settings is not None else Settings()
        if not isinstance(self.settings, Settings):
            self.settings = Settings.from_reference(self.settings)
        self._dist = dist
        if dist is None:
            self.data = as_problem(data)
        else:
            from .parallel import ShardProblem
            if not isinstance(data, ShardProblem):  # a whole problem as one shard
                d = as_problem(data)
                data = ShardProblem(d.A.colptr, d.A.rowidx, d.A.vals, d.b, d.c, d.spec, 0, d.m)
            self.data = data
        self._lib = native.load()
        self._h = None
        t0 = time.perf_counter()
        self._create()
        # mirror of EmbeddingCache.cg_iters_total (embedding.py:43,112): the
        # setup solve of g, then every solve's CG iterations; updated after
        # every step, so an on_iteration callback reads it like the reference's
        # ws.cache.cg_iters_total
        self.cache = _CacheView(native.query(self._h, native.Q_CG_ITERS_TOTAL))
        self.setup_time = time.perf_counter() - t0
        self.last_setup_time = self.setup_time
        self._final = None
        self._final_iter = None
        self._scal = None

    @property
    def sharded(self):
        return self._dist is not None

    # -- native plumbing ------------------------------------------------------
    def _arrays(self):
        d = self.data
        if self._dist is None:
            A = d.A
            return (A.nrows, A.ncols, A.colptr, A.rowidx, A.vals, d.b, d.c, d.spec, 0, 0)
        return (d.m, d.n, d.colptr, d.rowidx, d.vals, d.b, d.c, d.spec, d.row_lo, d.m_global)

    def _create(self):
        st = self.settings
        m, n, colptr, rowidx, vals, b, c, spec, row_lo, m_global = self._arrays()
        self._keep = [native.i64(colptr), native.i64(rowidx), native.f64(vals),
                      native.f64(b), native.f64(c), native.i64(spec.soc_dims),
                      native.i64(spec.psd_sides)]
        cp, ri, va, bb, cc, q, s = self._keep
        P = native.Problem(
            m=m, n=n, colptr=native.ptr(cp, native.i64p),
            rowidx=native.ptr(ri, native.i64p), vals=native.ptr(va), b=native.ptr(bb),
            c=native.ptr(cc), z=spec.zero_dim, l=spec.nonneg_dim, nq=q.size,
            q=native.ptr(q, native.i64p), ns=s.size, s=native.ptr(s, native.i64p),
            ep=spec.exp_dim, m_global=m_global, row_lo=row_lo)
        S = native.SettingsC(
            alpha=st.alpha, max_iters=st.max_iters, eps_pri=st.eps_pri, eps_dual=st.eps_dual,
            eps_gap=st.eps_gap, eps_infeas=st.eps_infeas, eps_unbdd=st.eps_unbdd,
            check_interval=st.check_interval, cg_max=st.cg_max,
            cg_tol=st.cg_tol if st.cg_tol is not None else 0.0,
            normalize=int(bool(st.normalize)), sweeps=st.sweeps, device=st.device,
            fast=(1 if getattr(st, "precond", False) else 0) | (2 if st.fast else 0))
        dist = None
        if self._dist is not None:
            sp = self._dist
            self._bounds = native.i64(sp.bounds)
            self._nid = None
            flags = 1 if sp.force else 0
            if getattr(sp, "host_name", None):
                nm = sp.host_name.encode()
                if len(nm) > 127:
                    raise ValueError("shared-memory group name longer than 127 bytes")
                self._nid = (native.C.c_uint8 * 128).from_buffer_copy(nm.ljust(128, b"\0"))
                flags |= 2
            elif sp.nccl_id is not None:
                self._nid = (native.C.c_uint8 * 128).from_buffer_copy(bytes(sp.nccl_id))
            dist = native.Dist(
                rank=sp.rank, world=sp.world,
                nccl_id=native.C.cast(self._nid, native.C.POINTER(native.C.c_uint8))
                if self._nid is not None else None,
                emu_group=sp.emu_group, bounds=native.ptr(self._bounds, native.i64p),
                flags=flags)
        h = native.C.c_void_p()
        rc = self._lib.scs_create(native.C.byref(P), native.C.byref(S),
                                  native.C.byref(dist) if dist is not None else None,
                                  native.C.byref(h))
        self._keep = None
        if rc != native.SCS_OK:
            try:
                native.check(rc, None)
            except native.NativeError as exc:
                _raise(exc, setup=True)
        self._h = h

    def allreduce(self, *vals):
        """Sum scalars over the shards (identity without sharding)."""
        arr = np.array(vals, dtype=np.float64)
        if self._dist is not None:
            self._call(self._lib.scs_allreduce(self._h, native.ptr(arr), arr.size))
        return arr

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.scs_destroy(h)
            except Exception:
                pass
            self._h = None

    def _call(self, rc):
        if rc != native.SCS_OK:
            try:
                native.check(rc, self._h)
            except native.NativeError as exc:
                _raise(exc)

    @property
    def scal(self) -> ScalingData:
        if self._scal is None:
            D = np.empty(self.data.m)
            E = np.empty(self.data.n)
            sg, rh = native.C.c_double(), native.C.c_double()
            self._call(self._lib.scs_get_scaling(self._h, native.ptr(D), native.ptr(E),
                                                 native.C.byref(sg), native.C.byref(rh)))
            self._scal = ScalingData(D, E, sg.value, rh.value)
        return self._scal

    def state(self):
        ln = self.data.n + self.data.m + 1
        u, v = np.empty(ln), np.empty(ln)
        self._call(self._lib.scs_get_state(self._h, native.ptr(u), native.ptr(v)))
        return u, v

    def apply_a(self, x, transpose=False):
        """A_hat x (or A_hat^T y) on the device (equilibrated matrix)."""
        x = native.f64(x)
        out = np.empty(self.data.n if transpose else self.data.m)
        self._call(self._lib.scs_apply_a(self._h, int(transpose), native.ptr(x), native.ptr(out)))
        return out

    # -- public API -----------------------------------------------------------
    def update_vectors(self, b=None, c=None):
        """Replace b and/or c, keeping A, its transpose and D, E on device."""
        t0 = time.perf_counter()
        nb = None if b is None else native.f64(b)
        nc = None if c is None else native.f64(c)
        if self._dist is None:
            self.data = ProblemData(self.data.A, self.data.b if nb is None else nb,
                                    self.data.c if nc is None else nc, self.data.spec)
        else:
            if nb is not None:
                self.data.b = nb
            if nc is not None:
                self.data.c = nc
        self._scal = None
        self._call(self._lib.scs_update_vectors(self._h, native.ptr(nb), native.ptr(nc)))
        self.cache.cg_iters_total = native.query(self._h, native.Q_CG_ITERS_TOTAL)
        self.last_setup_time = time.perf_counter() - t0
        return self.last_setup_time

    def solve(self, warm_start=None, on_iteration=None):
        """Workspace.solve (solver.py:336-378); the loop runs on the GPU."""
        st = self.settings
        n, m = self.data.n, self.data.m
        t0 = time.perf_counter()
        wx = wy = ws = None
        if warm_start is not None:
            x0, y0, s0 = (native.f64(t) for t in warm_start)
            if x0.shape != (n,) or y0.shape != (m,) or s0.shape != (m,):
                raise ValueError("warm start dimensions do not match the problem")
            wx, wy, ws = x0, y0, s0
        info = native.Info()
        if on_iteration is None:
            self._call(self._lib.scs_solve(self._h, native.ptr(wx), native.ptr(wy),
                                           native.ptr(ws), native.C.byref(info)))
        else:
            self._call(self._lib.scs_begin(self._h, native.ptr(wx), native.ptr(wy),
                                           native.ptr(ws)))
            # the termination check of iteration k runs inside step k+1 (it
            # shares that step's first matrix passes); a step that ends in
            # a status leaves the state -- and the iteration count -- at k
            while True:
                prev = int(info.iterations)
                self._call(self._lib.scs_step(self._h, 1, native.C.byref(info)))
                self.cache.cg_iters_total = int(info.cg_iters)
                if info.iterations > prev:
                    u, v = self.state()
                    on_iteration(SolverState(u=u, v=v, iter=int(info.iterations)))
                if info.status >= 0 or info.iterations >= st.max_iters or \
                        info.iterations == prev:
                    break
            self._call(self._lib.scs_finish(self._h, native.C.byref(info)))
        self.cache.cg_iters_total = int(info.cg_iters)
        status = _STATUS_BY_CODE[int(info.status)]
        res = Residuals(*[float(x) for x in info.res])
        self._final = None
        self._final_iter = int(info.iterations)
        if status in (Status.SOLVED, Status.MAX_ITERS_REACHED):
            sol = self._extract_point(status)
        else:
            u, v = self.state()
            self._final = SolverState(u=u, v=v, iter=self._final_iter)
            sol = self._extract(u, v, status)
        sol.info.iterations = int(info.iterations)
        sol.info.residuals = res
        sol.info.setup_time = self.last_setup_time
        sol.info.solve_time = time.perf_counter() - t0
        sol.info.cg_iters = int(info.cg_iters)
        self.launches = int(info.launches)
        return sol

    @property
    def final_state(self):
        """(u, v, iter) after the last solve (solver.py:374), fetched from the
        device on first access."""
        if self._final is None and self._final_iter is not None:
            u, v = self.state()
            self._final = SolverState(u=u, v=v, iter=self._final_iter)
        return self._final

    def _extract_point(self, status):
        """extract_solution (solver.py:251-270) for solved / max_iters_reached,
        on the device (scs_extract_point): x, y, s, objectives and point
        residuals without copying u, v out and the point back in."""
        d = self.data
        sol = Solution(status=status)
        # page-locked (pooled) result buffers: the device-to-host copies run at
        # link speed, overlapped with the point residuals
        x, y, s = native.pinned_empty(d.n), native.pinned_empty(d.m), native.pinned_empty(d.m)
        out = np.empty(5)
        self._call(self._lib.scs_extract_point(self._h, native.ptr(x), native.ptr(y),
                                               native.ptr(s), native.ptr(out)))
        sol.x, sol.y, sol.s = x, y, s  # y, s: this shard's rows when sharded
        sol.primal_obj = float(out[3])
        sol.dual_obj = float(-out[4])
        sol.info.pri_res, sol.info.dual_res, sol.info.gap = (float(t) for t in out[:3])
        return sol

    def point_residuals(self, x, y, s):
        out = np.empty(3)
        xs = [native.f64(t) for t in (x, y, s)]
        self._call(self._lib.scs_point_residuals(self._h, *[native.ptr(t) for t in xs],
                                                 native.ptr(out)))
        return tuple(float(t) for t in out)

    def _extract(self, u, v, status):
        """extract_solution (solver.py:251-288)."""
        d = self.data
        n, m = d.n, d.m
        sc = self.scal
        ux, uy, ut, vs = u[:n], u[n:n + m], u[-1], v[n:n + m]
        sol = Solution(status=status)
        if status in (Status.SOLVED, Status.MAX_ITERS_REACHED):
            x = sc.E * (ux / ut) / sc.sigma
            s = (vs / ut) / (sc.D * sc.sigma)
            y = sc.D * (uy / ut) / sc.rho
            sol.x, sol.y, sol.s = x, y, s  # y, s: this shard's rows when sharded
            sol.primal_obj = float(d.c @ x)
            sol.dual_obj = float(-self.allreduce(d.b @ y)[0])
            sol.info.pri_res, sol.info.dual_res, sol.info.gap = self.point_residuals(x, y, s)
        if status in (Status.INFEASIBLE, Status.INFEASIBLE_AND_UNBOUNDED):
            y_dir = sc.D * uy / sc.rho
            sol.certificate = y_dir / (-self.allreduce(d.b @ y_dir)[0])
            sol.primal_obj = np.inf
            sol.dual_obj = np.inf
        if status in (Status.UNBOUNDED, Status.INFEASIBLE_AND_UNBOUNDED):
            x_dir = sc.E * ux / sc.sigma
            ray = x_dir / (-(d.c @ x_dir))
            if status is Status.UNBOUNDED:
                sol.certificate = ray
                sol.primal_obj = -np.inf
                sol.dual_obj = -np.inf
            else:
                sol.certificate_unbounded = ray
        return sol


def solve(data_or_A, *args, settings=None):
    """``solve(data, settings=None)`` (solver.py:381-385) or the north-star
    form ``solve(A, b, c, cone, settings=None)`` with A a SparseMatrix (or
    any CSC duck type) and cone a ConeSpec or dict {"z","l","q","s","ep"}."""
    if args and len(args) >= 3:
        b, c, cone = args[0], args[1], args[2]
        if len(args) > 3:
            settings = args[3]
        data = ProblemData(SparseMatrix.from_any(data_or_A), b, c, ConeSpec.from_any(cone))
    else:
        data = data_or_A
        if args:
            settings = args[0]
    settings = settings if settings is not None else Settings()
    if not isinstance(settings, Settings):
        settings = Settings.from_reference(settings)
    ws = Workspace(data, settings)
    return ws.solve(warm_start=settings.warm_start)


def _finite_or_none(x):
    x = float(x)
    return x if np.isfinite(x) else None


def solution_to_dict(sol):
    """fileio.py:123-140."""
    doc = {"status": sol.status.value}
    for name, vec in (("x", sol.x), ("y", sol.y), ("s", sol.s),
                      ("certificate", sol.certificate)):
        if vec is not None:
            doc[name] = np.asarray(vec, dtype=float).tolist()
    doc["info"] = {
        "iters": int(sol.info.iterations),
        "pri_res": _finite_or_none(sol.info.pri_res),
        "dual_res": _finite_or_none(sol.info.dual_res),
        "gap": _finite_or_none(sol.info.gap),
        "solve_time_ms": 1000.0 * sol.info.solve_time,
    }
    return doc
