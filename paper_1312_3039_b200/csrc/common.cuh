// common.cuh -- shared device helpers: launch geometry, warp/block
// reductions, the deterministic "last block finalises" grid reduction, and
// the device control block that carries the solver's scalars between
// kernels (so the host never synchronises inside the iteration loop).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#ifndef SCS_BLOCK
#define SCS_BLOCK 256
#endif

namespace scs {

constexpr int kBlock = SCS_BLOCK;
constexpr int kWarps = kBlock / 32;
constexpr int kMaxRed = 8;       // scalars per reduction
constexpr int kMaxGrid = 4096;   // partial slots per scalar

// Device error bits (mapped to SCS_* codes on the host).
enum : int {
  ERR_CG_NONFINITE = 1,   // sparse_linalg.py:266-267,480-481
  ERR_CG_CURVATURE = 2,   // sparse_linalg.py:276-277
  ERR_CONE_NONFINITE = 4, // cones.py:194-200
  ERR_JACOBI = 8,         // cones.py:164-167
  ERR_SCHED = 16,         // internal: iteration graph variant != refresh schedule
};

// Everything the iteration needs to branch on, kept in device memory.
// Single-writer discipline: a field is written by exactly one thread (the
// last block of a reduction kernel, or a one-thread kernel) and read by
// later kernels in stream order.
struct Ctl {
  // persistent across iterations of one solve
  long long iter;           // SolverState.iter
  long long k_sched;        // EmbeddingCache.iter_count (embedding.py:180)
  long long cg_iters_total; // EmbeddingCache.cg_iters_total
  long long max_iters;
  long long check_interval;
  int status;               // SCS_RUNNING or a Status
  int stop;                 // 1: every kernel of the iteration is a no-op
  int err;                  // ERR_* bits
  int warm_zero;            // cg_warm == 0 exactly (skip A cg_warm gather)
  int force_check;          // residual kernels run regardless of interval
  int check_now;            // unused (kept for layout)
  int check_pending;        // the last finished iteration is due a check
  int pad1;
  // per-iteration scalars
  double tol;               // CG tolerance of this iteration
  double rs;                // CG r'r carried between CG steps
  double cg_alpha, cg_beta;
  int cg_done, cg_it;       // CG finished flag / iterations this call
  double corr;              // (h'p)/denom (embedding.py:192)
  double denom;             // 1 + h'g (embedding.py:159)
  // settings mirrored on device
  double alpha;             // over-relaxation
  double cg_tol;            // <= 0: schedule
  double eps[5];            // pri, dual, gap, infeas, unbdd
  // residual constants (depend on b, c, D, E, sigma, rho only)
  double b_norm, c_norm, b_ref, c_ref, sigma, rho;
  double res[8];            // Residuals of the last check
  double sums[kMaxRed];     // last finished reduction (debug)
  unsigned int counter;     // last-block counter
  unsigned int pad2;
  // device-side loop (solver.cu build_loop_graph): iterations still to run,
  // iterations run by the last loop launch, and how many were refreshes
  long long loop_left, loop_done, loop_refresh;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int L>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction of K values (any block size up to 1024);
// result valid in every thread.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K]) {
  __shared__ double sh[K][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh[k][warp] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sh[k][w];
    v[k] = t;
  }
  __syncthreads();
}

// Grid reduction with a deterministic finish: every block writes its
// partials, the last block to arrive sums them in fixed order.  Returns
// true (in every thread of that block) for the last block, with `v`
// holding the grid totals.  `part` holds K * gridDim.x doubles.
template <int K>
__device__ __forceinline__ bool grid_sum_last(double (&v)[K], double* part,
                                              unsigned int* counter) {
  block_sum<K>(v);
  __shared__ int am_last;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[k * G + blockIdx.x] = v[k];
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == (unsigned int)(G - 1));
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    acc[k] = 0.0;
    for (int i = threadIdx.x; i < G; i += blockDim.x) acc[k] += __ldcg(part + k * G + i);
  }
  block_sum<K>(acc);
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = acc[k];
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

}  // namespace scs
