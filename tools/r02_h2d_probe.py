"""Host-to-device copy of large pageable numpy arrays: the library's staged
path (scs_create's h2d_staged, via a CSR-only Workspace setup timing is not
isolated, so this probes the primitives) vs cudaHostRegister of the caller's
pages + one direct copy.  8 GB arrays."""
import ctypes, time
import numpy as np

rt = None
for cand in ("/usr/local/cuda/lib64/libcudart.so", "libcudart.so", "libcudart.so.12"):
    try:
        rt = ctypes.CDLL(cand)
        break
    except OSError:
        continue
rt.cudaSetDevice(0)
n = 1 << 30  # 8 GB of float64
a = np.ones(n)
a[::4096] = 2.0  # touch
d = ctypes.c_void_p()
assert rt.cudaMalloc(ctypes.byref(d), ctypes.c_size_t(8 * n)) == 0
rt.cudaDeviceSynchronize()
for trial in range(2):
    t = time.perf_counter()
    assert rt.cudaMemcpy(d, ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(8 * n), 1) == 0
    print(f"pageable cudaMemcpy 8 GB: {time.perf_counter() - t:.3f} s", flush=True)
t = time.perf_counter()
assert rt.cudaHostRegister(ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(8 * n), 0) == 0
t1 = time.perf_counter()
assert rt.cudaMemcpy(d, ctypes.c_void_p(a.ctypes.data), ctypes.c_size_t(8 * n), 1) == 0
t2 = time.perf_counter()
rt.cudaHostUnregister(ctypes.c_void_p(a.ctypes.data))
t3 = time.perf_counter()
print(f"cudaHostRegister {t1 - t:.3f} s + copy {t2 - t1:.3f} s + unregister {t3 - t2:.3f} s", flush=True)
# pinned staging, the library's scheme: 2 x 64 MB pinned buffers, memcpy into them, async copies
import threading
buf = [ctypes.c_void_p(), ctypes.c_void_p()]
for b in buf:
    rt.cudaMallocHost(ctypes.byref(b), ctypes.c_size_t(64 << 20))
t = time.perf_counter()
chunk = 8 << 20  # doubles per 64 MB
ctypes.memmove  # single-threaded host copy for the estimate
k = 0
for off in range(0, n, chunk):
    m = min(chunk, n - off)
    ctypes.memmove(buf[k], a.ctypes.data + 8 * off, 8 * m)
    rt.cudaMemcpy(ctypes.c_void_p(d.value + 8 * off), buf[k], ctypes.c_size_t(8 * m), 1)
    k ^= 1
print(f"1-thread staged 8 GB (serial): {time.perf_counter() - t:.3f} s", flush=True)
