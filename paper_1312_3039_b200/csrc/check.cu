// check.cu -- device side of the independent solution checker
// (the reference's `conesplit check`, cli.py:163-269).
// Cone-membership margins of a stacked vector, one value per cone block in
// the reference's order (cli.py:174-199): zero -max|v| (primal only; the
// dual of the zero cone is free), nonnegative min v, second-order
// v0 - ||v[1:]||, PSD the minimum eigenvalue of the unpacked svec block
// (device Jacobi), and -- no reference -- exponential: minus the distance
// to the cone (0 inside).  The residual products (scs_check_products) are
// stateless device SpMVs of the unscaled CSC matrix, independent of any
// solver handle.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/scs_b200.h"
#include "common.cuh"
#include "cones.cuh"

namespace scs {
namespace {

constexpr int kCheckThreads = 1024;

__device__ double block_max(double v) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = -INFINITY;
  for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) t = fmax(t, sh[w]);
  __syncthreads();
  return t;
}

// zero (mode 0: -max|v|) or nonnegative (mode 1: min v) block, one CTA
__global__ void k_margin_lin(const double* v, long long off, long long len, int mode, double* out) {
  double acc = -INFINITY;
  for (long long i = threadIdx.x; i < len; i += blockDim.x)
    acc = fmax(acc, mode == 0 ? fabs(v[off + i]) : -v[off + i]);
  acc = block_max(acc);
  if (threadIdx.x == 0) *out = -acc;
}

// second-order cones: CTA per cone
__global__ void k_margin_soc(const double* v, const long long* off, const long long* len, int nq,
                             double* out) {
  for (int q = blockIdx.x; q < nq; q += gridDim.x) {
    double s[1] = {0.0};
    for (long long i = 1 + threadIdx.x; i < len[q]; i += blockDim.x) {
      const double x = v[off[q] + i];
      s[0] += x * x;
    }
    block_sum<1>(s);
    if (threadIdx.x == 0) out[q] = v[off[q]] - sqrt(s[0]);
  }
}

// PSD blocks: CTA per block, Jacobi in per-CTA global scratch
__global__ void k_margin_psd(const double* v, const long long* off, const int* side, int ns,
                             int max_side, double* scratch, int* err, double* out) {
  __shared__ double cs[128], sn[128], dpp[128], dqq[128];
  __shared__ int pp[128], qq[128];
  double* M = scratch + (size_t)2 * blockIdx.x * max_side * max_side;
  for (int b = blockIdx.x; b < ns; b += gridDim.x) {
    const int k = side[b];
    double* V = M + (size_t)k * k;
    const int len = k * (k + 1) / 2;
    for (int e = threadIdx.x; e < len; e += blockDim.x) {
      int i, j;
      svec_rc(e, k, i, j);
      const double x = v[off[b] + e];
      const double val = (i == j) ? x : x / 1.4142135623730951;  // cli.py:163-175
      M[i * k + j] = val;
      M[j * k + i] = val;
    }
    __syncthreads();
    const bool ok = block_jacobi(M, V, k, cs, sn, pp, qq, dpp, dqq);
    double lo = INFINITY;
    for (int t = threadIdx.x; t < k; t += blockDim.x) lo = fmin(lo, M[t * k + t]);
    lo = -block_max(-lo);
    if (threadIdx.x == 0) {
      out[b] = lo;
      if (!ok) atomicOr(err, 1);
    }
    __syncthreads();
  }
}

// exponential cones: thread per cone, -||v - Pi(v)|| (Pi onto K_exp, or K_exp* when dual)
__global__ void k_margin_exp(const double* v, long long off, long long ne, int dual, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long e = tid; e < ne; e += nt) {
    const double* x = v + off + 3 * e;
    double p[3];
    if (dual) exp_proj_dual(x, p);
    else exp_proj_primal(x[0], x[1], x[2], p);
    const double d0 = x[0] - p[0], d1 = x[1] - p[1], d2 = x[2] - p[2];
    out[e] = -sqrt(d0 * d0 + d1 * d1 + d2 * d2);
  }
}

// warp per row of a CSR (or per column of a CSC): out[r] = sum_k v[k] x[idx[k]]
__global__ void k_rowdot(const long long* ptr, const int* idx, const double* v, long long rows,
                         const double* x, double* out) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = w; r < rows; r += nw) {
    double s = 0.0;
    for (long long k = ptr[r] + lane; k < ptr[r + 1]; k += 32) s += v[k] * x[idx[k]];
    s = warp_sum(s);
    if (lane == 0) out[r] = s;
  }
}
__global__ void k_narrow(const int64_t* in, long long n, int* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = tid; i < n; i += (long long)gridDim.x * blockDim.x) out[i] = (int)in[i];
}
__global__ void k_cols(const long long* colptr, long long n, int* col) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long j = w; j < n; j += nw)
    for (long long k = colptr[j] + (threadIdx.x & 31); k < colptr[j + 1]; k += 32) col[k] = (int)j;
}
__global__ void k_ptr_from_sorted(const int* keys, long long nnz, long long rows, long long* rp) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = tid; i <= rows; i += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (keys[mid] < i) lo = mid + 1; else hi = mid;
    }
    rp[i] = lo;
  }
}
__global__ void k_permute(const int* perm, const int* col, const double* v, long long nnz, int* ci,
                          double* av) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long k = tid; k < nnz; k += (long long)gridDim.x * blockDim.x) {
    ci[k] = col[perm[k]];
    av[k] = v[perm[k]];
  }
}

struct Buf {
  std::vector<void*> ps;
  ~Buf() {
    for (void* p : ps) cudaFree(p);
  }
  template <class T>
  T* get(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    ps.push_back(p);
    return (T*)p;
  }
};

}  // namespace
}  // namespace scs

extern "C" {

int64_t scs_cone_margin_count(int64_t z, int64_t l, int64_t nq, int64_t ns, int64_t ep,
                              int32_t dual) {
  return (z > 0 && !dual ? 1 : 0) + (l > 0 ? 1 : 0) + nq + ns + ep;
}

int scs_cone_margins(const double* vec, int64_t m, int64_t z, int64_t l, int64_t nq,
                     const int64_t* q, int64_t ns, const int64_t* s, int64_t ep, int32_t dual,
                     int32_t device, double* out, int64_t nout) {
  using namespace scs;
  if (!vec || !out || m < 0 || z < 0 || l < 0 || nq < 0 || ns < 0 || ep < 0) return SCS_EINVAL;
  if ((nq && !q) || (ns && !s)) return SCS_EINVAL;
  if (nout != scs_cone_margin_count(z, l, nq, ns, ep, dual)) return SCS_EINVAL;
  std::vector<long long> qoff(nq), qlen(nq), soff(ns);
  std::vector<int> sside(ns);
  long long o = z + l;
  for (int64_t i = 0; i < nq; ++i) {
    if (q[i] < 1) return SCS_EINVAL;
    qoff[i] = o;
    qlen[i] = q[i];
    o += q[i];
  }
  int max_side = 1;
  for (int64_t i = 0; i < ns; ++i) {
    if (s[i] < 1 || s[i] > 255) return SCS_EINVAL;
    soff[i] = o;
    sside[i] = (int)s[i];
    max_side = std::max(max_side, (int)s[i]);
    o += s[i] * (s[i] + 1) / 2;
  }
  const long long exp_off = o;
  o += 3 * ep;
  if (o != m) return SCS_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SCS_ECUDA;
  Buf buf;
  double* dv = buf.get<double>(m);
  double* dout = buf.get<double>(nout);
  long long* dqo = buf.get<long long>(nq);
  long long* dql = buf.get<long long>(nq);
  long long* dso = buf.get<long long>(ns);
  int* dss = buf.get<int>(ns);
  int* derr = buf.get<int>(1);
  const int gp = (int)std::min<int64_t>(std::max<int64_t>(ns, 1), 148);
  double* scratch = buf.get<double>((size_t)2 * gp * max_side * max_side);
  if (!dv || !dout || !dqo || !dql || !dso || !dss || !derr || !scratch) return SCS_ENOMEM;
  cudaMemcpy(dv, vec, m * sizeof(double), cudaMemcpyHostToDevice);
  if (nq) {
    cudaMemcpy(dqo, qoff.data(), nq * sizeof(long long), cudaMemcpyHostToDevice);
    cudaMemcpy(dql, qlen.data(), nq * sizeof(long long), cudaMemcpyHostToDevice);
  }
  if (ns) {
    cudaMemcpy(dso, soff.data(), ns * sizeof(long long), cudaMemcpyHostToDevice);
    cudaMemcpy(dss, sside.data(), ns * sizeof(int), cudaMemcpyHostToDevice);
  }
  cudaMemset(derr, 0, sizeof(int));
  long long k = 0;
  if (z > 0 && !dual) k_margin_lin<<<1, kCheckThreads>>>(dv, 0, z, 0, dout + k++);
  if (l > 0) k_margin_lin<<<1, kCheckThreads>>>(dv, z, l, 1, dout + k++);
  if (nq) {
    k_margin_soc<<<(int)std::min<int64_t>(nq, 4096), 256>>>(dv, dqo, dql, (int)nq, dout + k);
    k += nq;
  }
  if (ns) {
    k_margin_psd<<<gp, 256>>>(dv, dso, dss, (int)ns, max_side, scratch, derr, dout + k);
    k += ns;
  }
  if (ep) {
    const int g = (int)std::min<int64_t>((ep + 255) / 256, 4096);
    k_margin_exp<<<g, 256>>>(dv, exp_off, ep, dual, dout + k);
  }
  cudaError_t e = cudaMemcpy(out, dout, nout * sizeof(double), cudaMemcpyDeviceToHost);
  int herr = 0;
  cudaMemcpy(&herr, derr, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return SCS_ECUDA;
  if (herr) return SCS_ENOCONV;
  return SCS_OK;
}

// Stateless device products for the checker: Ax = A x and Aty = A^T y of a
// CSC matrix (the reference SparseMatrix; cli.py:209-210 uses spmv/spmv_t).
// A^T y is a warp-per-column dot over the CSC; A x goes through a device
// transpose (stable radix sort of the row indices) and a warp-per-row dot,
// so both are deterministic.  Either output may be NULL.
int scs_check_products(int64_t m, int64_t n, const int64_t* colptr, const int64_t* rowidx,
                       const double* vals, const double* x, const double* y, double* Ax,
                       double* Aty, int32_t device) {
  using namespace scs;
  if (m < 0 || n < 0 || !colptr) return SCS_EINVAL;
  const long long nnz = colptr[n];
  if (nnz < 0 || nnz >= (1LL << 31) - 1 || m >= (1LL << 31) - 1) return SCS_EINVAL;
  if ((Ax && !x) || (Aty && !y) || (nnz && (!rowidx || !vals))) return SCS_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SCS_ECUDA;
  Buf buf;
  long long* cp = buf.get<long long>(n + 1);
  int64_t* ri64 = buf.get<int64_t>(nnz);
  int* ri = buf.get<int>(nnz);
  double* v = buf.get<double>(nnz);
  if (!cp || !ri64 || !ri || !v) return SCS_ENOMEM;
  cudaMemcpy(cp, colptr, (n + 1) * sizeof(long long), cudaMemcpyHostToDevice);
  if (nnz) {
    cudaMemcpy(ri64, rowidx, nnz * sizeof(int64_t), cudaMemcpyHostToDevice);
    cudaMemcpy(v, vals, nnz * sizeof(double), cudaMemcpyHostToDevice);
  }
  const int G = 148 * 8, T = 256;
  k_narrow<<<G, T>>>(ri64, nnz, ri);
  if (Aty) {
    double* dy = buf.get<double>(m);
    double* dout = buf.get<double>(n);
    if (!dy || !dout) return SCS_ENOMEM;
    cudaMemcpy(dy, y, m * sizeof(double), cudaMemcpyHostToDevice);
    k_rowdot<<<G, T>>>(cp, ri, v, n, dy, dout);
    if (cudaMemcpy(Aty, dout, n * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return SCS_ECUDA;
  }
  if (Ax) {
    double* dx = buf.get<double>(n);
    double* dout = buf.get<double>(m);
    long long* rp = buf.get<long long>(m + 1);
    int* col = buf.get<int>(nnz);
    int* keys = buf.get<int>(nnz);
    int* iota = buf.get<int>(nnz);
    int* perm = buf.get<int>(nnz);
    int* ci = buf.get<int>(nnz);
    double* av = buf.get<double>(nnz);
    if (!dx || !dout || !rp || !col || !keys || !iota || !perm || !ci || !av) return SCS_ENOMEM;
    cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice);
    k_cols<<<G, T>>>(cp, n, col);
    std::vector<int> h_iota(nnz);
    for (long long k = 0; k < nnz; ++k) h_iota[k] = (int)k;
    if (nnz) cudaMemcpy(iota, h_iota.data(), nnz * sizeof(int), cudaMemcpyHostToDevice);
    int bits = 1;
    while ((1LL << bits) < m) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int*)ri, keys, (const int*)iota, perm,
                                    (int)nnz, 0, bits);
    void* tmp = buf.get<char>(tb);
    if (!tmp) return SCS_ENOMEM;
    cub::DeviceRadixSort::SortPairs(tmp, tb, (const int*)ri, keys, (const int*)iota, perm, (int)nnz,
                                    0, bits);
    k_ptr_from_sorted<<<G, T>>>(keys, nnz, m, rp);
    k_permute<<<G, T>>>(perm, col, v, nnz, ci, av);
    k_rowdot<<<G, T>>>(rp, ci, av, m, dx, dout);
    if (cudaMemcpy(Ax, dout, m * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return SCS_ECUDA;
  }
  if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) return SCS_ECUDA;
  return SCS_OK;
}

}  // extern "C"
