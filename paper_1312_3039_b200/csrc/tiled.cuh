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

// Ordered list of the non-empty tiles of this CTA's slab range, built in
// parallel (ballot compaction + block prefix) into shared memory.
__device__ __forceinline__ int tile_list(const Tiled& T, long long tb0, int fsb, int s_lo,
                                         int s_hi, unsigned short* list, int* wcount) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int total = 0;
  for (int base = s_lo; base < s_hi; base += blockDim.x) {
    const int s = base + tid;
    bool ne = false;
    if (s < s_hi) {
      const long long tb = tb0 + (long long)s * kTileNsub;
      ne = __ldg(T.ts + tb) != __ldg(T.ts + tb + fsb);
    }
    const unsigned mask = __ballot_sync(0xffffffffu, ne);
    if (lane == 0) wcount[warp] = __popc(mask);
    __syncthreads();
    int before = 0, all = 0;
    for (int w = 0; w < nw; ++w) {
      const int cw = wcount[w];
      if (w < warp) before += cw;
      all += cw;
    }
    if (ne) list[total + before + __popc(mask & ((1u << lane) - 1))] = (unsigned short)(s - s_lo);
    total += all;
    __syncthreads();
  }
  return total;
}

// Boundary runs of the 32 warps (rows nondecreasing in warp order, equal
// rows adjacent) folded into the accumulators by warp 0 with one segmented
// scan: deterministic, no serial loop.
template <int NV>
__device__ __forceinline__ void merge_bounds(const int* bndr, const double* bndv, double* acc) {
  const int lane = threadIdx.x & 31;
  int r1 = bndr[2 * lane], r2 = bndr[2 * lane + 1];
  double v1[NV], v2[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) { v1[t] = bndv[(2 * lane) * NV + t]; v2[t] = bndv[(2 * lane + 1) * NV + t]; }
  if (r2 == r1) {  // one run: everything is in slot 1
#pragma unroll
    for (int t = 0; t < NV; ++t) v1[t] += v2[t];
    r2 = -4;
  }
  // lane item = (head run r1, tail run r2 or r1)
  const bool two = r2 >= 0;
  const int tr = two ? r2 : r1;
  double ts[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) ts[t] = two ? v2[t] : v1[t];
  const int ptr = __shfl_up_sync(0xffffffffu, tr, 1);
  bool f = two || lane == 0 || ptr != tr;
  double v[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) v[t] = ts[t];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const bool fp = __shfl_up_sync(0xffffffffu, f, o);
    double vp[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) vp[t] = __shfl_up_sync(0xffffffffu, v[t], o);
    if (lane >= o && !f) {
#pragma unroll
      for (int t = 0; t < NV; ++t) v[t] += vp[t];
      f = fp;
    }
  }
  double carry[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) carry[t] = __shfl_up_sync(0xffffffffu, v[t], 1);
  const int nhr = __shfl_down_sync(0xffffffffu, r1, 1);
  if (two && r1 >= 0) {
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[(size_t)r1 * NV + t] += v1[t] + ((lane > 0 && ptr == r1) ? carry[t] : 0.0);
  }
  if (tr >= 0 && (lane == 31 || nhr != tr)) {
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[(size_t)tr * NV + t] += v[t];
  }
}

template <int NV, int STRIDE, class Epi>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tiled(Tiled T, Epi epi0, int sub, int splits, double* P) {
  Epi epi = epi0;
  if (!epi.load()) return;
  extern __shared__ double sm[];
  double* slabs = sm;                       // 2 x W * NV (double buffer)
  double* acc = sm + 2 * (size_t)T.W * NV;  // rows of this CTA * NV
  __shared__ int bndr[2 * (kTileThreads / 32)];
  __shared__ double bndv[2 * (kTileThreads / 32) * NV];
  __shared__ int wcount[kTileThreads / 32];
  unsigned short* tlist = reinterpret_cast<unsigned short*>(acc + (size_t)(T.RB / sub) * NV);
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
  const int ntl = tile_list(T, tb0, fsb, s_lo, s_hi, tlist, wcount);
  int li = 0;
  int s = ntl > 0 ? s_lo + tlist[0] : s_hi;
  if (s < s_hi) slab_of(s, slabs);
  int cur = 0;
  while (s < s_hi) {
    ++li;
    const int sn = li < ntl ? s_lo + tlist[li] : s_hi;
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
    // warp w owns the 4-aligned entry run [ws, we) of the (4-padded) tile;
    // rows it shares with neighbouring warps go to its boundary slots
    // (only min(nw, groups) warps take work, so no empty range sits between
    // two warps that share a row -- the merge scan relies on that)
    const long long q4 = (e1 - e0) >> 2;
    const long long na = q4 < nw ? q4 : nw;
    const long long ws = warp < na ? e0 + 4 * (q4 * warp / na) : e1;
    const long long we = warp < na ? e0 + 4 * (q4 * (warp + 1) / na) : e1;
    int fr = -2, lr = -3;
    if (we > ws) {
      const unsigned pf = __ldg(T.pk + ws) >> 16, pl = __ldg(T.pk + we - 1) >> 16;
      fr = pf == 0xffffu ? -2 : (int)pf - rel0;
      lr = pl == 0xffffu ? -3 : (int)pl - rel0;
    }
    if (lane == 0) {
      bndr[warp * 2] = fr;
      bndr[warp * 2 + 1] = lr;
#pragma unroll
      for (int t = 0; t < NV; ++t) { bndv[(warp * 2) * NV + t] = 0.0; bndv[(warp * 2 + 1) * NV + t] = 0.0; }
    }
    __syncwarp();
    auto emit = [&](int r, const double* v) {
      if (r < 0) return;
      double* dst = r == fr ? bndv + (warp * 2) * NV : (r == lr ? bndv + (warp * 2 + 1) * NV
                                                                 : acc + (size_t)r * NV);
#pragma unroll
      for (int t = 0; t < NV; ++t) dst[t] += v[t];
    };
    for (long long e = ws; e < we; e += 128) {
      const long long kb = e + 4 * lane;  // this lane's 4 contiguous entries
      unsigned p[4];
      double a[4];
      if (kb + 3 < we) {
        const uint4 pv = __ldcs(reinterpret_cast<const uint4*>(T.pk + kb));
        p[0] = pv.x; p[1] = pv.y; p[2] = pv.z; p[3] = pv.w;
        double d0, d1, d2, d3;
        asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(d0), "=d"(d1), "=d"(d2), "=d"(d3) : "l"(T.v + kb));
        a[0] = d0; a[1] = d1; a[2] = d2; a[3] = d3;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { p[k] = 0xffff0000u; a[k] = 0.0; }
      }
      int r[4];
      double x[4][NV];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned rr = p[k] >> 16;
        const bool ok = rr != 0xffffu;
        r[k] = ok ? (int)rr - rel0 : -1 - (lane * 4 + k);  // padding: unique, never matches
        const int c = (int)(p[k] & 0xffffu);
#pragma unroll
        for (int t = 0; t < NV; ++t) x[k][t] = ok ? a[k] * slab[c * NV + t] : 0.0;
      }
      // lane-local folding: head run, closed middle runs (emitted), tail run
      double hs[NV], ts[NV];
#pragma unroll
      for (int t = 0; t < NV; ++t) hs[t] = x[0][t];
      const int hr = r[0];
      int k = 1;
#pragma unroll
      for (int kk = 1; kk < 4; ++kk)
        if (k == kk && r[kk] == hr) {
#pragma unroll
          for (int t = 0; t < NV; ++t) hs[t] += x[kk][t];
          ++k;
        }
      const bool single = k == 4;
      int tr = hr;
#pragma unroll
      for (int t = 0; t < NV; ++t) ts[t] = hs[t];
      if (!single) {
        tr = r[k];
#pragma unroll
        for (int t = 0; t < NV; ++t) ts[t] = 0.0;
#pragma unroll
        for (int kk = 1; kk < 4; ++kk) {
          if (kk < k) continue;
          if (r[kk] != tr) {  // run [.., kk) closed inside this lane
            emit(tr, ts);
            tr = r[kk];
#pragma unroll
            for (int t = 0; t < NV; ++t) ts[t] = 0.0;
          }
#pragma unroll
          for (int t = 0; t < NV; ++t) ts[t] += x[kk][t];
        }
      }
      // warp segmented scan of the tail runs: a single-run lane continues
      // the previous lane's tail run when the rows match
      const int ptr = __shfl_up_sync(0xffffffffu, tr, 1);
      bool f = !single || lane == 0 || ptr != tr;
      double v[NV];
#pragma unroll
      for (int t = 0; t < NV; ++t) v[t] = ts[t];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const bool fp = __shfl_up_sync(0xffffffffu, f, o);
        double vp[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) vp[t] = __shfl_up_sync(0xffffffffu, v[t], o);
        if (lane >= o && !f) {
#pragma unroll
          for (int t = 0; t < NV; ++t) v[t] += vp[t];
          f = fp;
        }
      }
      // head run of a multi-run lane closes with the carry of the lanes before
      double carry[NV];
#pragma unroll
      for (int t = 0; t < NV; ++t) carry[t] = __shfl_up_sync(0xffffffffu, v[t], 1);
      const int nhr = __shfl_down_sync(0xffffffffu, hr, 1);
      if (!single) {
        double tot[NV];
#pragma unroll
        for (int t = 0; t < NV; ++t) tot[t] = hs[t] + ((lane > 0 && ptr == hr) ? carry[t] : 0.0);
        emit(hr, tot);
      }
      // tail run ends here unless the next lane starts with the same row
      if (lane == 31 || nhr != tr) emit(tr, v);
      __syncwarp();
    }
    __syncthreads();  // everyone is done with slab `cur` before it is refilled
    if (warp == 0) merge_bounds<NV>(bndr, bndv, acc);  // warp-order fold of shared rows
    __syncthreads();
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

// scatter sorted entry k into its 4-padded sub-tile position
__global__ void k_tile_pack(const int* perm, const int* skey, const long long* ts_raw,
                            const long long* ts_pad, const int* rowid, const int* ci,
                            const double* v, long long nnz, int RB, int W, unsigned* pk,
                            double* tv) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt) {
    const int s = perm[k];
    const int t = skey[k];
    const long long pos = ts_pad[t] + (k - ts_raw[t]);
    pk[pos] = ((unsigned)(rowid[s] % RB) << 16) | (unsigned)(ci[s] % W);
    tv[pos] = v[s];
  }
}
__global__ void k_fill_pad(unsigned* pk, double* tv, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < n; k += nt) { pk[k] = 0xffff0000u; tv[k] = 0.0; }
}
__global__ void k_pad4(const long long* ts_raw, long long ntile, long long* cnt) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long t = tid; t < ntile; t += nt) cnt[t] = (ts_raw[t + 1] - ts_raw[t] + 3) & ~3LL;
}

}  // namespace scs
