"""Problem and solution files.

Two formats, chosen by the file suffix:

* ``.json`` -- the reference's single-document JSON (fileio.py:1-13,
  problem_to_dict :57-75, problem_from_dict :78-110, solution_to_dict
  :123-140, solution_from_dict :143-167), with the same member names,
  the same ``FileFormatError(member, message)`` (a ValueError, :26-31) and
  shortest round-trip float text, so problem and solution files move between
  the two packages unchanged.  The optional ``"ep"`` cone member carries the
  exponential-cone count (no reference) and is written only when
  nonzero.
* ``.scsb`` -- a binary CSC layout for instances JSON cannot hold (10^8-10^9
  nonzeros).  Little-endian; a 128-byte header

      magic  b"SCSB\\x01\\x00\\x00\\x00"
      int64  m, n, nnz, z, l, ep, nq, ns, idx_bytes (4 or 8), 0, 0, 0, 0, 0, 0

  followed by the arrays, each starting on an 8-byte boundary:
  q[nq] int64, s[ns] int64, colptr[n+1] int64, rowidx[nnz] int32|int64,
  vals[nnz] float64, b[m] float64, c[n] float64.  Reading maps the file
  (numpy memmap): nothing is parsed, and `Workspace` copies the arrays to
  the device straight from the page cache.
"""

import json
import os

import numpy as np

from .api import ConeSpec, ProblemData, Solution, SolveInfo, SparseMatrix, Status
from .api import solution_to_dict

MAGIC = b"SCSB\x01\x00\x00\x00"
HEADER_BYTES = 128


class FileFormatError(ValueError):
    """Malformed document; `member` names the offending field (fileio.py:26-31)."""

    def __init__(self, member, message):
        super().__init__(f"{member}: {message}")
        self.member = member


def _require(doc, member, kind):
    # fileio.py:34-54
    if member not in doc:
        raise FileFormatError(member, "missing member")
    value = doc[member]
    if kind == "int":
        if not isinstance(value, int) or isinstance(value, bool):
            raise FileFormatError(member, "expected an integer")
    elif kind == "object":
        if not isinstance(value, dict):
            raise FileFormatError(member, "expected an object")
    elif kind == "int_array":
        if not isinstance(value, list) or any(
                not isinstance(v, int) or isinstance(v, bool) for v in value):
            raise FileFormatError(member, "expected an array of integers")
    elif kind == "num_array":
        if not isinstance(value, list) or any(
                not isinstance(v, (int, float)) or isinstance(v, bool) for v in value):
            raise FileFormatError(member, "expected an array of numbers")
    return value


def problem_to_dict(data):
    spec = data.spec
    cone = {"z": int(spec.zero_dim), "l": int(spec.nonneg_dim),
            "q": [int(v) for v in spec.soc_dims], "s": [int(v) for v in spec.psd_sides]}
    if spec.exp_dim:
        cone["ep"] = int(spec.exp_dim)
    return {
        "m": int(data.m),
        "n": int(data.n),
        "A": {"colptr": np.asarray(data.A.colptr).tolist(),
              "rowidx": np.asarray(data.A.rowidx).tolist(),
              "vals": np.asarray(data.A.vals, dtype=float).tolist()},
        "b": np.asarray(data.b, dtype=float).tolist(),
        "c": np.asarray(data.c, dtype=float).tolist(),
        "cone": cone,
    }


def problem_from_dict(doc):
    if not isinstance(doc, dict):
        raise FileFormatError("<document>", "expected a JSON object")
    m = _require(doc, "m", "int")
    n = _require(doc, "n", "int")
    a_doc = _require(doc, "A", "object")
    colptr = _require(a_doc, "colptr", "int_array")
    rowidx = _require(a_doc, "rowidx", "int_array")
    vals = _require(a_doc, "vals", "num_array")
    b = _require(doc, "b", "num_array")
    c = _require(doc, "c", "num_array")
    cone = _require(doc, "cone", "object")
    z = _require(cone, "z", "int")
    l = _require(cone, "l", "int")
    q = _require(cone, "q", "int_array")
    s = _require(cone, "s", "int_array")
    ep = _require(cone, "ep", "int") if "ep" in cone else 0
    try:
        A = SparseMatrix(m, n, np.asarray(colptr, dtype=np.int64),
                         np.asarray(rowidx, dtype=np.int64), np.asarray(vals, dtype=float))
    except ValueError as exc:
        raise FileFormatError("A", str(exc)) from exc
    try:
        spec = ConeSpec(z, l, tuple(q), tuple(s), ep)
    except ValueError as exc:
        raise FileFormatError("cone", str(exc)) from exc
    try:
        return ProblemData(A, np.asarray(b, dtype=float), np.asarray(c, dtype=float), spec)
    except ValueError as exc:
        raise FileFormatError("b/c/cone", str(exc)) from exc


def _vector_field(doc, member, expected_len):
    # fileio.py:113-119
    if member not in doc or doc[member] is None:
        return None
    arr = _require(doc, member, "num_array")
    if expected_len is not None and len(arr) != expected_len:
        raise FileFormatError(member, f"expected length {expected_len}, got {len(arr)}")
    return np.asarray(arr, dtype=float)


def solution_from_dict(doc):
    # fileio.py:143-167
    if not isinstance(doc, dict):
        raise FileFormatError("<document>", "expected a JSON object")
    status_str = doc.get("status")
    try:
        status = Status(status_str)
    except ValueError:
        raise FileFormatError("status", f"unknown status {status_str!r}") from None
    info = doc.get("info", {})
    if not isinstance(info, dict):
        raise FileFormatError("info", "expected an object")
    sinfo = SolveInfo(
        iterations=int(info.get("iters", 0)),
        pri_res=np.nan if info.get("pri_res") is None else float(info["pri_res"]),
        dual_res=np.nan if info.get("dual_res") is None else float(info["dual_res"]),
        gap=np.nan if info.get("gap") is None else float(info["gap"]),
        solve_time=float(info.get("solve_time_ms", 0.0)) / 1000.0)
    sol = Solution(status=status, info=sinfo)
    sol.x = _vector_field(doc, "x", None)
    sol.y = _vector_field(doc, "y", None)
    sol.s = _vector_field(doc, "s", None)
    sol.certificate = _vector_field(doc, "certificate", None)
    return sol


def _dump(doc, path):
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")


def _load(path):
    try:
        with open(path) as fh:
            return json.load(fh)
    except json.JSONDecodeError as exc:
        raise FileFormatError("<document>", f"invalid JSON: {exc}") from exc


# --- binary CSC (.scsb) -----------------------------------------------------

def _align8(x):
    return (x + 7) & ~7


def write_problem_binary(path, data):
    A = data.A
    colptr = np.ascontiguousarray(A.colptr, dtype=np.int64)
    nnz = int(colptr[-1]) if colptr.size else 0
    idx_t = np.int32 if data.m < 2**31 else np.int64
    rowidx = np.ascontiguousarray(np.asarray(A.rowidx)[:nnz], dtype=idx_t)
    spec = data.spec
    q = np.asarray(spec.soc_dims, dtype=np.int64)
    s = np.asarray(spec.psd_sides, dtype=np.int64)
    hdr = np.zeros(15, dtype=np.int64)
    hdr[:9] = [data.m, data.n, nnz, spec.zero_dim, spec.nonneg_dim, spec.exp_dim, q.size, s.size,
               np.dtype(idx_t).itemsize]
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(hdr.tobytes())
        for arr in (q, s, colptr, rowidx, np.asarray(A.vals[:nnz], dtype=np.float64),
                    np.asarray(data.b, dtype=np.float64), np.asarray(data.c, dtype=np.float64)):
            arr = np.ascontiguousarray(arr)
            arr.tofile(fh)
            pad = _align8(arr.nbytes) - arr.nbytes
            if pad:
                fh.write(b"\0" * pad)


def read_problem_binary(path, mmap=True):
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(HEADER_BYTES)
    if len(head) < HEADER_BYTES or head[:8] != MAGIC:
        raise FileFormatError("<header>", "not an SCSB problem file")
    hdr = np.frombuffer(head[8:], dtype=np.int64)
    m, n, nnz, z, l, ep, nq, ns, ib = (int(v) for v in hdr[:9])
    if min(m, n, nnz, z, l, ep, nq, ns) < 0 or ib not in (4, 8):
        raise FileFormatError("<header>", "negative size or bad index width")
    layout = [("q", np.int64, nq), ("s", np.int64, ns), ("colptr", np.int64, n + 1),
              ("rowidx", np.int32 if ib == 4 else np.int64, nnz), ("vals", np.float64, nnz),
              ("b", np.float64, m), ("c", np.float64, n)]
    need = HEADER_BYTES + sum(_align8(np.dtype(t).itemsize * k) for _, t, k in layout)
    if size < need:
        raise FileFormatError("<document>", f"truncated: {size} bytes, expected {need}")
    arrs, off = {}, HEADER_BYTES
    for name, t, k in layout:
        if mmap and k:
            arrs[name] = np.memmap(path, dtype=t, mode="r", offset=off, shape=(k,))
        else:
            with open(path, "rb") as fh:
                fh.seek(off)
                arrs[name] = np.fromfile(fh, dtype=t, count=k)
        off += _align8(np.dtype(t).itemsize * k)
    try:
        A = SparseMatrix(m, n, arrs["colptr"], arrs["rowidx"], arrs["vals"])
    except ValueError as exc:
        raise FileFormatError("A", str(exc)) from exc
    try:
        spec = ConeSpec(z, l, tuple(int(v) for v in arrs["q"]),
                        tuple(int(v) for v in arrs["s"]), ep)
    except ValueError as exc:
        raise FileFormatError("cone", str(exc)) from exc
    try:
        return ProblemData(A, arrs["b"], arrs["c"], spec)
    except ValueError as exc:
        raise FileFormatError("b/c/cone", str(exc)) from exc


# --- suffix dispatch (fileio.py:182-195) -------------------------------------

def _binary(path):
    return str(path).endswith(".scsb")


def write_problem(path, data):
    if _binary(path):
        write_problem_binary(path, data)
    else:
        _dump(problem_to_dict(data), path)


def read_problem(path):
    if _binary(path):
        return read_problem_binary(path)
    return problem_from_dict(_load(path))


def write_solution(path, sol):
    _dump(solution_to_dict(sol), path)


def read_solution(path):
    return solution_from_dict(_load(path))
