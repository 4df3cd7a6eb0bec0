// tiled.cuh -- slab-tiled SpMV: gathers from shared memory.
//
// ncu on the CSR kernels (profiles/r01_ncu_c3_spmv_v1.txt) shows they are
// bound by the L1->L2 request rate, not by DRAM: every random gather of
// x[col] is one 32-byte sector request for 8 useful bytes.  This kernel
// removes the gathers from the memory system:
//
//  * the matrix is re-laid out once (after equilibration) into tiles
//    (row block of RB rows) x (column slab of W columns), each split into
//    kTileNsub row sub-tiles.  Inside a sub-tile the row segments are
//    sorted by length and grouped 32 to a chunk (SELL-C-sigma with C = 32,
//    sigma = the sub-tile); a chunk stores its entries column-interleaved
//    (step k of all 32 lanes contiguous): fp64 value + 16-bit column
//    offset, 10 bytes per nonzero, plus one 16-bit row id per lane;
//  * a CTA owns a row block (or part of one) and walks the column slabs of
//    its range: it stages the slab of the gather vector in shared memory
//    with cp.async (double-buffered; L2 traffic ~ |x| per row block instead
//    of 32 B per nonzero); each lane then sums one row segment in registers
//    -- coalesced 256 B value / 64 B column loads per step, gathers from
//    shared memory, no shuffles -- and adds it to its row's shared
//    accumulator (each row has one segment per sub-tile, so the update is
//    exclusive and the order of a row's partial sums is fixed: the result
//    is deterministic);
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
  const long long* cs;          // (NB * S) * kTileNsub + 1: first chunk of each sub-tile
  const long long* co;          // nchunk + 1: first entry of each chunk (32 * width each)
  const unsigned short* rid;    // 32 per chunk: row - block start, 0xffff = idle lane
  const unsigned short* col;    // per entry: column - slab start
  const double* v;              // per entry value (0 for padding)
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
      ne = __ldg(T.cs + tb) != __ldg(T.cs + tb + fsb);
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

template <int NV, int STRIDE, class Epi>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tiled(Tiled T, Epi epi0, int sub, int splits, double* P) {
  Epi epi = epi0;
  if (!epi.load()) return;
  extern __shared__ double sm[];
  double* slabs = sm;                       // 2 x W * NV (double buffer)
  double* acc = sm + 2 * (size_t)T.W * NV;  // rows of this CTA * NV
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
    const long long c_lo = __ldg(T.cs + tb), c_hi = __ldg(T.cs + tb + fsb);
    for (long long ch = c_lo + warp; ch < c_hi; ch += nw) {
      const long long off = __ldg(T.co + ch);
      const int wid = (int)((__ldg(T.co + ch + 1) - off) >> 5);
      const unsigned rr = __ldg(T.rid + ch * 32 + lane);
      const double* vp = T.v + off + lane;
      const unsigned short* cp = T.col + off + lane;
      double sum[NV];
#pragma unroll
      for (int t = 0; t < NV; ++t) sum[t] = 0.0;
      int k = 0;
      for (; k + 4 <= wid; k += 4) {  // four steps of the chunk in flight
        double a[4];
        int c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { a[u] = __ldcs(vp + (k + u) * 32); c[u] = __ldcs(cp + (k + u) * 32); }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int t = 0; t < NV; ++t) sum[t] = fma(a[u], slab[c[u] * NV + t], sum[t]);
      }
      for (; k < wid; ++k) {
        const double a = __ldcs(vp + k * 32);
        const int c = __ldcs(cp + k * 32);
#pragma unroll
        for (int t = 0; t < NV; ++t) sum[t] = fma(a, slab[c * NV + t], sum[t]);
      }
      if (rr != 0xffffu) {
        const int r = (int)rr - rel0;  // one segment per row per sub-tile: exclusive
#pragma unroll
        for (int t = 0; t < NV; ++t) acc[(size_t)r * NV + t] += sum[t];
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

// --- SELL-style sub-tile layout ---------------------------------------------
// entries are already sorted by sub-tile (stable: row-major inside)
__global__ void k_seg_flags(const int* skey, const int* perm, const int* rowid, long long nnz,
                            int* flag) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt)
    flag[k] = (k == 0 || skey[k] != skey[k - 1] || rowid[perm[k]] != rowid[perm[k - 1]]) ? 1 : 0;
}
// seg_start[seg] = first entry of each row segment (flag prefix sum = seg + 1)
__global__ void k_seg_starts(const int* flag, const int* incl, long long nnz, long long* seg_start) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt)
    if (flag[k]) seg_start[incl[k] - 1] = k;
}
// sort key of a segment: (sub-tile, length descending)
__global__ void k_seg_keys(const long long* seg_start, long long nseg, long long nnz,
                           const int* skey, unsigned long long* key2, int* tile_of) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long q = tid; q < nseg; q += nt) {
    const long long a = seg_start[q], b = q + 1 < nseg ? seg_start[q + 1] : nnz;
    const int t = skey[a];
    tile_of[q] = t;
    key2[q] = ((unsigned long long)t << 20) | (unsigned long long)((1 << 20) - 1 - (b - a));
  }
}
// chunks per sub-tile from the (sorted) segment counts
__global__ void k_tile_chunks(const long long* tss, long long ntile, long long* nch) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long t = tid; t < ntile; t += nt) nch[t] = (tss[t + 1] - tss[t] + 31) / 32;
}
// entries per chunk = 32 * length of its first (longest) segment
__global__ void k_chunk_sizes(const long long* tss, const long long* cs, long long ntile,
                              const int* order, const long long* seg_start, long long nseg,
                              long long nnz, long long* csz) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long t = tid; t < ntile; t += nt) {
    for (long long c = cs[t]; c < cs[t + 1]; ++c) {
      const long long p = tss[t] + (c - cs[t]) * 32;
      const long long q = order[p];
      const long long len = (q + 1 < nseg ? seg_start[q + 1] : nnz) - seg_start[q];
      csz[c] = 32 * len;
    }
  }
}
__global__ void k_sell_scatter(const long long* tss, const long long* cs, const long long* co,
                               const int* order, const int* tile_sorted,
                               const long long* seg_start, long long nseg, long long nnz,
                               const int* perm, const int* rowid, const int* ci, const double* v,
                               int RB, int W, unsigned short* rid, unsigned short* col,
                               double* tv) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long p = tid; p < nseg; p += nt) {
    const int t = tile_sorted[p];
    const long long pos = p - tss[t];
    const long long c = cs[t] + pos / 32;
    const int lane = (int)(pos % 32);
    const long long q = order[p];
    const long long a = seg_start[q], b = q + 1 < nseg ? seg_start[q + 1] : nnz;
    rid[c * 32 + lane] = (unsigned short)(rowid[perm[a]] % RB);
    const long long base = co[c] + lane;
    for (long long e = a; e < b; ++e) {
      const int s = perm[e];
      col[base + (e - a) * 32] = (unsigned short)(ci[s] % W);
      tv[base + (e - a) * 32] = v[s];
    }
  }
}
__global__ void k_fill_u16(unsigned short* x, long long n, unsigned short val) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) x[i] = val;
}

}  // namespace scs
