"""Build the native library in-tree: paper_1312_3039_b200/libscs_b200.so.

    python -m paper_1312_3039_b200.build [--verbose]

nvcc cross-compiles for sm_100a without a GPU.  The library links the CUDA
runtime statically and NCCL dynamically (row sharding over NVLink).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libscs_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["solver.cu", "check.cu", "host_gen.cpp"]
HEADERS = ["common.cuh", "cones.cuh", "kernels.cuh", "stream.cuh"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _nccl_flags():
    inc = "/usr/include/nccl.h"
    for libdir in ("/usr/lib/x86_64-linux-gnu", "/usr/local/cuda/lib64"):
        if os.path.exists(os.path.join(libdir, "libnccl.so")) and os.path.exists(inc):
            return ["-DSCS_WITH_NCCL", f"-L{libdir}", "-lnccl"]
    return []


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "scs_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = _nvcc()
    nccl = _nccl_flags()
    objs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo"]
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *common, *ARCH, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
            cmd += [f for f in nccl if f.startswith("-D")]
        else:
            cmd += ["-Xcompiler", "-pthread", "-Xcompiler", "-ffp-contract=off"]
        _run(cmd, verbose)
        objs.append(obj)
    link = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
            *[f for f in nccl if not f.startswith("-D")], "-Xcompiler", "-pthread"]
    _run(link, verbose)
    for o in objs:
        os.remove(o)
    return LIB


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
