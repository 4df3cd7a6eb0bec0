// tiled.cuh -- slab-tiled SpMV: gathers from shared memory.
//
// ncu on the CSR kernels (profiles/r01_ncu_c3_spmv_v1.txt) shows they are
// bound by the L1->L2 request rate, not by DRAM: every random gather of
// x[col] is one 32-byte sector request for 8 useful bytes.  This kernel
// removes the gathers from the memory system:
//
//  * the matrix is re-laid out once (after equilibration) into tiles
//    (row block of RB rows) x (column slab of W columns); a tile's entries
//    are contiguous, in row-major order, each stored as a packed
//    (row - block start, col - slab start) pair of 16-bit offsets plus the
//    fp64 value: 12 bytes per nonzero, as CSR;
//  * a CTA owns a row block (or a quarter of one) and walks the column
//    slabs of its range: it stages the slab of the gather vector in shared
//    memory with coalesced loads (L2 traffic ~ |x| per row block instead of
//    32 B per nonzero), then each warp streams a row-aligned, contiguous run
//    of the tile's entries, gathers from shared memory, and folds the
//    products into per-row shared accumulators with a warp segmented scan
//    (rows are contiguous runs, so each row's partial sums are combined in
//    a fixed order: the result is deterministic);
//  * after the last slab the CTA runs the same per-row epilogue (Epi::row)
//    as the CSR kernel, coalesced, or -- when the slab range is split over
//    several CTAs to fill the GPU -- writes per-split partial rows that
//    k_tiled_combine sums in split order before the epilogue.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace scs {

constexpr int kTileThreads = 1024;
constexpr int kTileNsub = 4;  // row sub-blocks per format row block

struct Tiled {
  long long rows, cols;
  int RB, W, S, NB;             // rows per block, columns per slab, #slabs, #blocks
  const long long* ts;          // (NB * S) * kTileNsub + 1 sub-tile starts
  const unsigned* pk;           // (row_rel << 16) | col_rel
  const double* v;
};

// First entry >= pos (within [e0, e1)) that starts a new row, so that warps
// own whole rows of the tile.
__device__ __forceinline__ long long row_align(const unsigned* __restrict__ pk, long long pos,
                                               long long e0, long long e1) {
  if (pos <= e0) return e0;
  if (pos >= e1) return e1;
  const unsigned rprev = __ldg(pk + pos - 1) >> 16;
  const int lane = threadIdx.x & 31;
  for (long long q = pos; q < e1; q += 32) {
    const long long k = q + lane;
    const bool start = k < e1 && (__ldg(pk + k) >> 16) != rprev;
    const unsigned mask = __ballot_sync(0xffffffffu, start);
    if (mask) return q + __ffs(mask) - 1;
  }
  return e1;
}

// async copy of one gather-vector slab (NV values per column) into smem
template <int NV, int STRIDE>
__device__ __forceinline__ void slab_issue(const double* __restrict__ xb, long long c0, int wc,
                                           double* dst) {
  for (int i = threadIdx.x; i < wc; i += blockDim.x) {
    const double* src = xb + (size_t)(c0 + i) * STRIDE;
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst + (size_t)i * NV);
    if constexpr (NV == 1) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src));
    } else {
      static_assert(NV == 2, "tiled NV");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
    }
  }
  asm volatile("cp.async.commit_group;");
}

__device__ __forceinline__ int next_tile(const Tiled& T, long long tb0, int fsb, int s, int s_hi) {
  for (; s < s_hi; ++s) {
    const long long tb = tb0 + (long long)s * kTileNsub;
    if (__ldg(T.ts + tb) != __ldg(T.ts + tb + fsb)) return s;
  }
  return s_hi;
}

template <int NV, int STRIDE, class Epi>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tiled(Tiled T, Epi epi0, int sub, int splits, double* P) {
  Epi epi = epi0;
  if (!epi.load()) return;
  extern __shared__ double sm[];
  double* slabs = sm;                       // 2 x W * NV (double buffer)
  double* acc = sm + 2 * (size_t)T.W * NV;  // rows of this CTA * NV
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int sp = blockIdx.x % splits;
  const int rest = blockIdx.x / splits;
  const int sbc = rest % sub, b = rest / sub;
  const int fsb = kTileNsub / sub;          // format sub-blocks per CTA
  const int rsub = T.RB / kTileNsub;
  const int rel0 = sbc * fsb * rsub;
  const long long r0 = (long long)b * T.RB + rel0;
  const long long left = T.rows - r0;
  const int R = left <= 0 ? 0 : (int)(left < (long long)fsb * rsub ? left : (long long)fsb * rsub);
  for (int i = tid; i < R * NV; i += blockDim.x) acc[i] = 0.0;
  const int s_lo = (int)((long long)T.S * sp / splits), s_hi = (int)((long long)T.S * (sp + 1) / splits);
  const long long tb0 = (long long)b * T.S * kTileNsub + (long long)sbc * fsb;
  auto slab_of = [&](int s, double* dst) {
    const long long c0 = (long long)s * T.W;
    const int wc = (int)((T.cols - c0) < T.W ? (T.cols - c0) : T.W);
    slab_issue<NV, STRIDE>(epi.xb, c0, wc, dst);
  };
  int s = next_tile(T, tb0, fsb, s_lo, s_hi);
  if (s < s_hi) slab_of(s, slabs);
  int cur = 0;
  while (s < s_hi) {
    const int sn = next_tile(T, tb0, fsb, s + 1, s_hi);
    if (sn < s_hi) {
      slab_of(sn, slabs + (size_t)(cur ^ 1) * T.W * NV);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();  // slab s visible to the whole CTA
    const double* slab = slabs + (size_t)cur * T.W * NV;
    const long long tb = tb0 + (long long)s * kTileNsub;
    const long long e0 = __ldg(T.ts + tb), e1 = __ldg(T.ts + tb + fsb);
    const long long len = e1 - e0;
    const long long ws = row_align(T.pk, e0 + len * warp / nw, e0, e1);
    const long long we = row_align(T.pk, e0 + len * (warp + 1) / nw, e0, e1);
    for (long long e = ws; e < we; e += 128) {
      // four chunks of the stream in flight before any use
      unsigned p[4];
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long k = e + u * 32 + lane;
        const bool ok = k < we;
        p[u] = ok ? __ldcs(T.pk + k) : 0u;
        a[u] = ok ? __ldcs(T.v + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (e + u * 32 >= we) break;  // warp-uniform
        const bool ok = e + u * 32 + lane < we;
        const int r = ok ? (int)(p[u] >> 16) - rel0 : -1 - lane;
        const int c = (int)(p[u] & 0xffffu);
        double x[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) x[t] = ok ? a[u] * slab[c * NV + t] : 0.0;
        // segmented inclusive scan over lanes of equal row (runs are contiguous)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int rp = __shfl_up_sync(0xffffffffu, r, o);
#pragma unroll
          for (int t = 0; t < NV; ++t) {
            const double xp = __shfl_up_sync(0xffffffffu, x[t], o);
            if (lane >= o && rp == r) x[t] += xp;
          }
        }
        const int rn = __shfl_down_sync(0xffffffffu, r, 1);
        if (ok && (lane == 31 || rn != r)) {
#pragma unroll
          for (int t = 0; t < NV; ++t) acc[r * NV + t] += x[t];
        }
        __syncwarp();
      }
    }
    __syncthreads();  // everyone is done with slab `cur` before it is refilled
    cur ^= 1;
    s = sn;
  }
  __syncthreads();
  constexpr int NR = Epi::NR > 0 ? Epi::NR : 1;
  if (splits > 1) {
    for (int i = tid; i < R; i += blockDim.x)
#pragma unroll
      for (int t = 0; t < NV; ++t) P[((long long)sp * T.rows + r0 + i) * NV + t] = acc[i * NV + t];
    return;
  }
  double red[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) red[t] = 0.0;
  for (int i = tid; i < R; i += blockDim.x) {
    typename Epi::Pre pre;
    epi.pre(r0 + i, pre);
    double sv[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) sv[t] = acc[i * NV + t];
    epi.row(r0 + i, sv, pre, red);
  }
  epi.extra(red);
  if constexpr (Epi::NR > 0) {
    if (grid_sum_last<Epi::NR>(red, epi.V.part, &epi.V.ctl->counter)) {
      if (epi.defer) {
        if (threadIdx.x == 0)
          for (int t = 0; t < Epi::NR; ++t) epi.V.dred[t] = red[t];
      } else {
        epi.finish(red);
      }
    }
  }
}

// Sum the per-split partial rows in split order, then the epilogue.
template <class Epi>
__global__ void __launch_bounds__(kBlock) k_tiled_combine(const double* P, int splits, long long rows,
                                                          Epi epi0) {
  Epi epi = epi0;
  if (!epi.load()) return;
  constexpr int NV = Epi::NV;
  constexpr int NR = Epi::NR > 0 ? Epi::NR : 1;
  double red[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) red[t] = 0.0;
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  for (long long j = tid; j < rows; j += nt) {
    typename Epi::Pre pre;
    epi.pre(j, pre);
    double s[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) s[t] = 0.0;
    for (int sp = 0; sp < splits; ++sp)
#pragma unroll
      for (int t = 0; t < NV; ++t) s[t] += P[((long long)sp * rows + j) * NV + t];
    epi.row(j, s, pre, red);
  }
  epi.extra(red);
  if constexpr (Epi::NR > 0) {
    if (grid_sum_last<Epi::NR>(red, epi.V.part, &epi.V.ctl->counter)) {
      if (epi.defer) {
        if (threadIdx.x == 0)
          for (int t = 0; t < Epi::NR; ++t) epi.V.dred[t] = red[t];
      } else {
        epi.finish(red);
      }
    }
  }
}

// ---- format build (setup) ----------------------------------------------------
__global__ void k_expand_rows(const long long* rp, long long rows, int* out) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = w; r < rows; r += nw)
    for (long long k = rp[r] + lane; k < rp[r + 1]; k += 32) out[k] = (int)r;
}

// sort key: ((block, slab), sub-block); entries keep CSR order within a key
__global__ void k_tile_keys(const int* rowid, const int* ci, long long nnz, int RB, int W, int S,
                            int* key) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const int rsub = RB / kTileNsub;
  for (long long k = tid; k < nnz; k += nt) {
    const int r = rowid[k], c = ci[k];
    key[k] = (((r / RB) * S + c / W) * kTileNsub) + (r % RB) / rsub;
  }
}

__global__ void k_tile_pack(const int* perm, const int* rowid, const int* ci, const double* v,
                            long long nnz, int RB, int W, unsigned* pk, double* tv) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt) {
    const int s = perm[k];
    pk[k] = ((unsigned)(rowid[s] % RB) << 16) | (unsigned)(ci[s] % W);
    tv[k] = v[s];
  }
}

}  // namespace scs
