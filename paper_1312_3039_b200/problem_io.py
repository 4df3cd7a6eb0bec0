"""Binary problem files: a CSC layout for instances the
reference's JSON documents cannot hold (10^8-10^9 nonzeros).
The reference's JSON problem/solution format (fileio.py) is out of scope
 and is not reimplemented here; the result dictionary of
``solution_to_dict`` (fileio.py:123-140) lives in ``api``.

``.scsb`` layout, little-endian; a 128-byte header

    magic  b"SCSB\\x01\\x00\\x00\\x00"
    int64  m, n, nnz, z, l, ep, nq, ns, idx_bytes (4 or 8), 0, 0, 0, 0, 0, 0

followed by the arrays, each starting on an 8-byte boundary:
q[nq] int64, s[ns] int64, colptr[n+1] int64, rowidx[nnz] int32|int64,
vals[nnz] float64, b[m] float64, c[n] float64.  Reading maps the file
(numpy memmap) instead of parsing it.  Building the ``SparseMatrix`` still
makes one O(nnz) pass: int32 row indices are widened to the reference's
int64 layout (8 bytes per nonzero of host memory) and validated
(sparse_linalg.py:34-54).
"""

import os

import numpy as np

from .api import ConeSpec, ProblemData, SparseMatrix

MAGIC = b"SCSB\x01\x00\x00\x00"
HEADER_BYTES = 128


class FileFormatError(ValueError):
    """Malformed file; `member` names the offending field (the convention
    of the reference's fileio.FileFormatError)."""

    def __init__(self, member, message):
        super().__init__(f"{member}: {message}")
        self.member = member


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


def _binary(path):
    return str(path).endswith(".scsb")


def write_problem(path, data):
    """Write a ``.scsb`` problem file."""
    if not _binary(path):
        raise ValueError("problem files are binary .scsb here; the reference's JSON documents "
                         "are read and written by conesplit.fileio")
    write_problem_binary(path, data)


def read_problem(path):
    """Read a ``.scsb`` problem file (memory-mapped)."""
    if not _binary(path):
        raise ValueError("problem files are binary .scsb here; the reference's JSON documents "
                         "are read and written by conesplit.fileio")
    return read_problem_binary(path)
