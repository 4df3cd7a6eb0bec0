// stream.cuh -- TMA-streamed slab-tiled SpMV (sm_100a).
//
// Why: the CSR kernels are bound by the L2 slice throughput, not by HBM --
// every random gather x[col] costs a 32-byte sector for 8-16 useful bytes
// (config 5: 32 GB of gather sectors + 12 GB of matrix per pass,
// profiles/r01_ncu_c5_spmv_banded.txt).  r01's slab-tiled kernel (retired
// in r02) moved the gathers into shared memory but loaded the matrix
// with ordinary per-chunk loads whose latency it could not cover at
// config 5's ~1-2 entries per row segment.  This kernel keeps the idea and
// moves every byte of the matrix and of the gathered vector with the
// Tensor Memory Accelerator's bulk copies into a multi-stage shared-memory
// ring, so the consumers never touch global memory in the inner loop:
//
//  * format (built once, after equilibration): rows in sub-blocks of
//    kStmRS = 4096 rows = 16 warp sections of 256 rows; columns in slabs of
//    W columns.  A tile = (sub-block, slab).  Inside a warp section the row
//    entries are placed on 32 lanes x D steps: the rows 32 j + l of a
//    section are pinned to lane l (overflow entries go to free slots of
//    other lanes, k_stm_pin), step k of all 32 lanes is contiguous.  Every
//    tile is cut into pieces of at most `cap` bytes (a piece = a step range
//    of every section; normally the whole tile) and each
//    piece is one contiguous blob: header, owner table, fp64 values, u16
//    slot words (column - slab start | j << 12 | overflow << 15).  Sub-
//    blocks whose tiles are too sparse to pay
//    for a slab load (config 5: A^T rows of the t-variables, two entries
//    each) stay CSR units, computed from the CSR arrays by the consumers;
//  * schedule (host, at setup): a unit = one sub-block (or, with
//    SCS_STREAM_PAIR=1, a pair of sub-blocks sharing the slab loads of an
//    NV = 1 pass), optionally split over slab
//    ranges when there are too few units for 148 SMs; units are placed on
//    persistent CTAs by longest-processing-time first, and each CTA gets a
//    flat command list (one command per piece, in order);
//  * kernel: one producer warp walks the command list and issues, per
//    stage, the bulk copy of the piece and -- when the slab changes -- of
//    the slab of the gathered vector (double-buffered) onto a full
//    mbarrier with expect_tx; 16 consumer warps wait on it, each walks its
//    own section four steps at a time and adds every product into the
//    shared accumulator of its row (the rows of a step are distinct, so the
//    updates need no atomics and their order is fixed -- deterministic),
//    then releases the stage on an empty mbarrier.
//    At the end of a unit each warp runs the pass's per-row epilogue
//    (Epi::row) over its own rows -- or writes split partials that
//    k_split_combine sums in split order -- and the CTA's reductions go
//    through the usual deterministic grid_sum_last.
//  (r02: 4096-column slabs with a 12-bit column field, a local search over
//  slot placement, whole-tile pieces; DESIGN.md §5.1 has the measurements.)
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace scs {

constexpr int kStmRS = 4096;        // rows per sub-block
constexpr int kStmSecRows = 256;    // rows per warp section
constexpr int kStmWarps = kStmRS / kStmSecRows;  // 16 consumer warps
constexpr int kStmThreads = (kStmWarps + 1) * 32;
constexpr int kStmHdr = 48;         // piece header bytes: u32 nslots, u16 wsec[17]
constexpr int kStmOwn = 32 * 16;    // + per warp section, per lane: owner lane of its overflow slots
constexpr int kStmData = kStmHdr + kStmOwn;  // values start here; then u16 slot words
constexpr int kStmMaxW = 4096;      // slot word column field: 12 bits
__host__ __device__ constexpr unsigned long long stm_piece_bytes(unsigned long long ns) {
  return kStmData + 10ULL * ns;
}
constexpr int kStmMaxStages = 8;

enum : unsigned short { STM_END = 1, STM_CSR = 2, STM_PAIR = 4, STM_TILE = 8, STM_CSR32 = 16 };

struct StmCmd {
  unsigned long long off;  // blob byte offset
  unsigned bytes;          // blob bytes (0: header-only stage)
  unsigned slab;
  long long row0;          // first row of the unit
  unsigned short flags;
  unsigned char half;      // sub-block within a pair unit
  unsigned char sp;        // split index (raw partial slot)
  unsigned pad;
};
static_assert(sizeof(StmCmd) == 32, "StmCmd layout");

struct Stm {
  long long rows, cols;
  int W, S, NB, cap;
  const unsigned char* blob;
};

struct StmCtl {  // per stage, written by the producer before its arrive
  long long row0;
  unsigned short flags;
  unsigned char half, sp;
  int xbuf;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-issuing the probe, leaving
// issue slots (and power, under the sustained power cap) to the working warps
constexpr unsigned kStmSuspendNs = 2000;
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "STM_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra STM_WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity), "r"(kStmSuspendNs)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, unsigned bytes,
                                               unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Epilogue (or raw split partials) for the rows of this warp's section,
// reading and clearing the shared accumulator `a` (NV per row).
template <int NV, class Epi>
__device__ __forceinline__ void stm_rows(Epi& epi, double* a, long long r0, int cnt, int splits,
                                         int sp, long long rows, double* P, double* red) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kStmSecRows; i += 32) {
    double sv[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) { sv[t] = a[i * NV + t]; a[i * NV + t] = 0.0; }
    if (i < cnt) {
      const long long row = r0 + i;
      if (splits > 1) {
#pragma unroll
        for (int t = 0; t < NV; ++t) P[((long long)sp * rows + row) * NV + t] = sv[t];
      } else {
        typename Epi::Pre pre;
        epi.pre(row, pre);
        epi.row(row, sv, pre, red);
      }
    }
  }
}

// One warp section of a piece.  Slot word (16 bits): column in the slab
// (12 bits) | j << 12 (3 bits) | overflow << 15.  A pinned entry's row is
// owned by its lane (local row = 32 j + lane), so the pinned read-modify-
// writes of a step hit 32 distinct rows in the minimum number of shared-
// memory wavefronts; overflow entries (in another lane's free slots) share
// the same update: all overflow entries of one owner lane sit in one lane,
// and k_stm_pin keeps them off the steps where the owner lane holds the
// same row, so the rows of a step are always distinct.  Padding slots hold
// value 0 (word: column = lane, pinned, j = 0): the update is predicated on
// a nonzero value, which skips them -- and explicit zeros, whose products
// add nothing to a row sum (x + 0 = x, 0 + -0 = 0).
template <int NV, int STRIDE, int U, bool MASK>
__device__ __forceinline__ void stm_steps(const double* vals, const unsigned short* idx, int k,
                                          int k1, const double* xs, double* a, unsigned own) {
  const int lane = threadIdx.x & 31;
  double pr[U][NV];
  unsigned rw[U];
  bool live[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {  // every load of the batch before its stores
    live[u] = false;
    rw[u] = 0;
#pragma unroll
    for (int t = 0; t < NV; ++t) pr[u][t] = 0.0;
    if (MASK && k + u >= k1) continue;  // warp-uniform: no load issued past the section's end
    const double v = vals[(k + u) * 32 + lane];
    const unsigned id = idx[(k + u) * 32 + lane];
    live[u] = v != 0.0;
    rw[u] = ((id >> 12) & 7u) << 5 | ((id >> 15) ? own : (unsigned)lane);
    const unsigned col = id & 0xfffu;
#pragma unroll
    for (int t = 0; t < NV; ++t) pr[u][t] = v * xs[col * STRIDE + t];
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (live[u])
#pragma unroll
      for (int t = 0; t < NV; ++t) a[rw[u] * NV + t] += pr[u][t];
}

// A warp's steps of one piece: batches of 4 steps, then the 1-3 left as one
// masked batch (sections hold ~4-9 steps per piece), so a section's tail
// keeps its loads in flight together instead of running step by step.
template <int NV, int STRIDE>
__device__ __forceinline__ void stm_piece(const double* vals, const unsigned short* idx, int k0,
                                          int k1, const double* xs, double* a, unsigned own) {
  int k = k0;
  for (; k + 4 <= k1; k += 4) stm_steps<NV, STRIDE, 4, false>(vals, idx, k, k1, xs, a, own);
  if (k < k1) stm_steps<NV, STRIDE, 3, true>(vals, idx, k, k1, xs, a, own);
}

// CSR unit rows [r0, rend) of this warp, L lanes per row (warp-uniform loop)
template <int L, int NV, int STRIDE, class Epi>
__device__ __forceinline__ void stm_csr(Epi& epi, const Csr& M, long long r0, long long rend,
                                        int splits, long long rows, double* P, double* red) {
  constexpr int G = 32 / L;
  const int lane = threadIdx.x & 31, gl = lane & (L - 1), gi = lane / L;
  for (long long rb = r0; rb < rend; rb += G) {
    const long long r = rb + gi;
    const bool ok = r < rend;
    long long k0 = 0, k1 = 0;
    if (ok) { k0 = __ldg(M.rp + r); k1 = __ldg(M.rp + r + 1); }
    double s[NV];
    row_dot<L, NV, STRIDE>(M, k0, k1, gl, epi.xb, s);
    if (ok && gl == 0) {
      if (splits > 1) {
        for (int q = 0; q < splits; ++q)
#pragma unroll
          for (int t = 0; t < NV; ++t) P[((long long)q * rows + r) * NV + t] = q == 0 ? s[t] : 0.0;
      } else {
        typename Epi::Pre pre;
        epi.pre(r, pre);
        epi.row(r, s, pre, red);
      }
    }
  }
}

template <int NV, int STRIDE, class Epi>
__global__ void __launch_bounds__(kStmThreads, 1)
    k_stream(Stm F, const StmCmd* __restrict__ cmds, const long long* __restrict__ coff, Csr M,
             Epi epi0, int splits, double* P, int NS, int NB, int accb) {
  Epi epi = epi0;
  if (!epi.load()) return;
  extern __shared__ __align__(128) unsigned char stm_sm[];
  double* acc = reinterpret_cast<double*>(stm_sm);
  const int xbytes = F.W * STRIDE * 8;
  // accb: accumulator bytes (sub-blocks per unit x 4096 rows x NV doubles)
  double* xbuf0 = reinterpret_cast<double*>(stm_sm + accb);
  unsigned char* stages = stm_sm + accb + NB * xbytes;  // NB = 2 (double-buffered) or 1 slab buffers
  unsigned long long* full = reinterpret_cast<unsigned long long*>(stages + (size_t)NS * F.cap);
  unsigned long long* empty = full + kStmMaxStages;
  StmCtl* sctl = reinterpret_cast<StmCtl*>(empty + kStmMaxStages);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < accb / 8; i += blockDim.x) acc[i] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kStmWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long c0 = coff[blockIdx.x], c1 = coff[blockIdx.x + 1];
  constexpr int NR = Epi::NR > 0 ? Epi::NR : 1;
  double red[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) red[t] = 0.0;

  if (warp == kStmWarps) {
    // ---------------- producer warp ----------------
    unsigned long long pol = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    long long slab_cur = -1;
    int xb = 1;
    long long last0 = -1, last1 = -1;  // last stage that read slab buffer 0 / 1
    int st = -1;
    unsigned ph = 1;
    for (long long base = c0; base < c1; base += 32) {
      StmCmd mine{};
      if (base + lane < c1) mine = cmds[base + lane];
      const int cnt = (int)(c1 - base < 32 ? c1 - base : 32);
      for (int j = 0; j < cnt; ++j) {
        const unsigned long long off = __shfl_sync(0xffffffffu, mine.off, j);
        const unsigned bytes = __shfl_sync(0xffffffffu, mine.bytes, j);
        const unsigned slab = __shfl_sync(0xffffffffu, mine.slab, j);
        const long long row0 = __shfl_sync(0xffffffffu, mine.row0, j);
        const unsigned fl = __shfl_sync(0xffffffffu, (unsigned)mine.flags | ((unsigned)mine.half << 16) |
                                                         ((unsigned)mine.sp << 24), j);
        const long long i = base - c0 + j;
        if (++st == NS) st = 0;
        if (st == 0) ph ^= 1u;
        if (i >= NS) mbar_wait(empty + st, ph ^ 1u);
        const bool tile = bytes > 0 && !(fl & STM_CSR);
        unsigned slab_bytes = 0;
        long long cstart = 0, jlast = -1;
        if (tile && (long long)slab != slab_cur) {
          if (NB == 2) xb ^= 1;
          else xb = 0;  // one buffer: wait below for the last stage that read it
          jlast = xb ? last1 : last0;
          slab_cur = slab;
          cstart = (long long)slab * F.W;
          const long long wc = F.cols - cstart < F.W ? F.cols - cstart : F.W;
          slab_bytes = (unsigned)(((wc * STRIDE * 8) + 15) & ~15LL);
        }
        if (tile) {
          if (xb) last1 = i; else last0 = i;
        }
        // the piece is issued as soon as its stage is free; the slab copy
        // (same full barrier) only once the slab buffer's last reader has
        // released it -- with one stage per slab, waiting for the buffer
        // before the piece would cap the ring at two pieces in flight
        if (lane == 0) {
          StmCtl c;
          c.row0 = row0;
          c.flags = (unsigned short)((fl & 0xffff) | (tile ? STM_TILE : 0));
          c.half = (unsigned char)((fl >> 16) & 0xff);
          c.sp = (unsigned char)(fl >> 24);
          c.xbuf = xb;
          sctl[st] = c;
          if (tile) {
            mbar_arrive_tx(full + st, slab_bytes + bytes);
            bulk_g2s(stages + (size_t)st * F.cap, F.blob + off, bytes, full + st, pol);
          } else {
            mbar_arrive(full + st);
          }
        }
        if (slab_bytes) {
          if (jlast >= 0 && jlast > i - NS) mbar_wait(empty + (int)(jlast % NS), (unsigned)((jlast / NS) & 1));
          if (lane == 0)
            bulk_g2s_plain(xbuf0 + (size_t)xb * (xbytes / 8), epi.xb + cstart * STRIDE, slab_bytes,
                           full + st);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- consumer warps ----------------
    const long long ncmd = c1 - c0;
    int st = -1;
    unsigned ph = 1;
    for (long long i = 0; i < ncmd; ++i) {
      if (++st == NS) st = 0;
      if (st == 0) ph ^= 1u;
      mbar_wait(full + st, ph);
      const StmCtl c = sctl[st];
      if (c.flags & STM_CSR) {
        // sparse sub-block straight from CSR: 4 lanes per row, or a warp per
        // row when its rows are long
        const long long r0 = c.row0 + (long long)warp * kStmSecRows;
        const long long rend = (r0 + kStmSecRows < F.rows) ? r0 + kStmSecRows : F.rows;
        if (c.flags & STM_CSR32)
          stm_csr<32, NV, STRIDE>(epi, M, r0, rend, splits, F.rows, P, red);
        else
          stm_csr<4, NV, STRIDE>(epi, M, r0, rend, splits, F.rows, P, red);
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        continue;
      }
      const unsigned char* blob = stages + (size_t)st * F.cap;
      if (c.flags & STM_TILE) {
        const unsigned nslots = *reinterpret_cast<const unsigned*>(blob);
        if (nslots) {
          const unsigned short* wsec = reinterpret_cast<const unsigned short*>(blob + 4);
          const int k0 = wsec[warp], k1 = wsec[warp + 1];
          const unsigned own = blob[kStmHdr + warp * 32 + lane];
          const double* vals = reinterpret_cast<const double*>(blob + kStmData);
          const unsigned short* idx =
              reinterpret_cast<const unsigned short*>(blob + kStmData + 8 * (size_t)nslots);
          const double* xs = xbuf0 + (size_t)c.xbuf * (xbytes / 8);
          double* a = acc + ((size_t)c.half * kStmRS + (size_t)warp * kStmSecRows) * NV;
          stm_piece<NV, STRIDE>(vals, idx, k0, k1, xs, a, own);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      if (c.flags & STM_END) {
        __syncwarp();  // this warp's accumulator updates are visible to all its lanes
        const int nsb = (c.flags & STM_PAIR) ? 2 : 1;
        for (int h = 0; h < nsb; ++h) {
          const long long r0 = c.row0 + (long long)h * kStmRS + (long long)warp * kStmSecRows;
          const long long left = F.rows - r0;
          const int cnt = left <= 0 ? 0 : (int)(left < kStmSecRows ? left : kStmSecRows);
          double* a = acc + ((size_t)h * kStmRS + (size_t)warp * kStmSecRows) * NV;
          stm_rows<NV>(epi, a, r0, cnt, splits, c.sp, F.rows, P, red);
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (splits > 1) return;  // k_split_combine runs the epilogue and the reductions
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
__global__ void __launch_bounds__(kBlock) k_split_combine(const double* P, int splits, long long rows,
                                                          long long r0, long long r1, Epi epi0) {
  Epi epi = epi0;
  if (!epi.load()) return;
  constexpr int NV = Epi::NV;
  constexpr int NR = Epi::NR > 0 ? Epi::NR : 1;
  double red[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) red[t] = 0.0;
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  for (long long j = r0 + tid; j < r1; j += nt) {  // rows [r0, r1) of `rows`
    typename Epi::Pre pre;
    epi.pre(j, pre);
    double s[NV];
#pragma unroll
    for (int t = 0; t < NV; ++t) s[t] = 0.0;
    // eight splits' loads in flight at a time, added in split order
    int sp = 0;
    for (; sp + 8 <= splits; sp += 8) {
      double v[8][NV];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int t = 0; t < NV; ++t) v[q][t] = __ldcs(P + ((long long)(sp + q) * rows + j) * NV + t);
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int t = 0; t < NV; ++t) s[t] += v[q][t];
    }
    for (; sp < splits; ++sp)
#pragma unroll
      for (int t = 0; t < NV; ++t) s[t] += __ldcs(P + ((long long)sp * rows + j) * NV + t);
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

__global__ void k_expand_rows(const long long* rp, long long rows, int* out) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = w; r < rows; r += nw)
    for (long long k = rp[r] + lane; k < rp[r + 1]; k += 32) out[k] = (int)r;
}

// ---- format build (setup) ----------------------------------------------------

// Sort key of every entry: warp section ((sub-block, slab) tile * 16 + warp),
// then the lane that owns its row (local row mod 32), then the bank of its
// gather word rotated by the lane -- so that in each step the 32 lanes tend
// to read different shared-memory banks of the slab.
__global__ void k_stm_keys(const int* rowid, const int* ci, long long nnz, int W, int S,
                           unsigned long long* key) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt) {
    const int r = rowid[k], c = ci[k];
    const long long sec = ((long long)(r / kStmRS) * S + c / W) * kStmWarps + (r % kStmRS) / kStmSecRows;
    const unsigned rl = (unsigned)(r % kStmSecRows), ln = rl & 31u;
    const unsigned bank = ((unsigned)(c % W) - ln) & 15u;
    key[k] = ((unsigned long long)sec << 12) | (ln << 7) | (bank << 3) | (rl >> 5);
  }
}
__global__ void k_stm_sec(const unsigned long long* key, long long nnz, int* sec) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt) sec[k] = (int)(key[k] >> 12);
}

// Slots of one section (one thread per section).  Depth D starts at
// ceil(E / 32); the i-th entry of owner lane l sits at step i of lane l
// while i < D (pinned; lanes that are not full start at step l mod D and
// wrap, which spreads the free slots over all steps).  The excess of each owner lane (largest first)
// takes free slots -- steps >= another lane's own count -- at pairwise
// distinct steps, so two overflow entries of one row never share a step;
// pinned entries of the owner are then swapped (key and perm, inside the
// owner's run) so that no step holds a pinned and an overflow entry of the
// same row.  A lane hosts the overflow of at most one owner (hown: the
// owner of each lane's overflow slots, so a slot word needs only the row's
// j = row >> 5).  D grows until this succeeds; sections deeper than kStmPinMax
// steps or 2 D0 + 16 (rows far longer than their neighbours) are flagged
// 0xffff and their sub-block becomes a CSR unit.
// slot = step * 32 + lane, | 1 << 30 for overflow.
constexpr int kStmPinMax = 128;
constexpr int kStmSearchMax = 24;  // local search on sections of at most this depth

// Modelled shared-memory wavefronts of one (step, half-warp) of a section:
// the gather (8-byte words: entries of one bank class col & 15 conflict;
// padding slots gather column = lane) plus twice the accumulator read-
// modify-write (rows of one class row & 15; padding is skipped).  Per
// (step, half) the class counts are kept as 16 packed 4-bit counters.
__device__ __forceinline__ int stm_nib_max(unsigned long long c) {
  int m = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) m = max(m, (int)((c >> (4 * b)) & 15ull));
  return m;
}
__device__ __forceinline__ unsigned long long stm_gbit(unsigned c, int l) {
  return 1ull << (4 * ((c >> 31) ? ((c >> 24) & 15u) : (unsigned)(l & 15)));
}
__device__ __forceinline__ unsigned long long stm_rbit(unsigned c) {
  return (c >> 31) ? 1ull << (4 * ((c >> 11) & 15u)) : 0ull;
}

// Local search after the greedy placement: within each lane, swap the
// contents of two steps (entries of the lane's own rows, hosted overflow
// entries, padding) when the rows of both steps stay distinct and the
// modelled wavefronts of the two steps drop.  On C5-like sections this
// lowers the gather conflicts by ~15% and the accumulator ones by ~5%
// (tools/stm_sim.cpp).  Grid cell: valid << 31 | class << 24 | row << 11 |
// entry.  Updates slot[] of the moved entries.
__device__ void stm_search(const unsigned long long* key, long long p0, long long E, int D, int* slot) {
  unsigned g[kStmSearchMax * 32];
  unsigned long long rows[kStmSearchMax][4], gc[kStmSearchMax][2], rc[kStmSearchMax][2];
  for (int i = 0; i < D * 32; ++i) g[i] = 0;
  for (int k = 0; k < D; ++k) {
    rows[k][0] = rows[k][1] = rows[k][2] = rows[k][3] = 0;
  }
  for (long long e = 0; e < E; ++e) {
    const unsigned long long kk = key[p0 + e];
    const unsigned row = (unsigned)(kk & 7u) * 32u + (unsigned)((kk >> 7) & 31u);
    const unsigned cls = (unsigned)(((kk >> 3) + (kk >> 7)) & 15u);
    const int sl = slot[p0 + e] & ((1 << 30) - 1);
    g[sl] = 1u << 31 | cls << 24 | row << 11 | (unsigned)e;
    rows[sl >> 5][row >> 6] |= 1ull << (row & 63);
  }
  for (int k = 0; k < D; ++k)
    for (int h = 0; h < 2; ++h) {
      unsigned long long a = 0, r = 0;
      for (int l = h * 16; l < h * 16 + 16; ++l) {
        a += stm_gbit(g[k * 32 + l], l);
        r += stm_rbit(g[k * 32 + l]);
      }
      gc[k][h] = a;
      rc[k][h] = r;
    }
  for (int pass = 0; pass < 2; ++pass) {
    bool any = false;
    for (int l = 0; l < 32; ++l) {
      const int h = l >> 4;
      for (int k1 = 0; k1 < D; ++k1)
        for (int k2 = k1 + 1; k2 < D; ++k2) {
          const unsigned a = g[k1 * 32 + l], b = g[k2 * 32 + l];
          if (!((a | b) >> 31)) continue;
          const unsigned ra = (a >> 11) & 255u, rb = (b >> 11) & 255u;
          // rows stay distinct: a's row absent from step k2, b's from k1
          if ((a >> 31) && ((rows[k2][ra >> 6] >> (ra & 63)) & 1ull)) continue;
          if ((b >> 31) && ((rows[k1][rb >> 6] >> (rb & 63)) & 1ull)) continue;
          const unsigned long long ga = stm_gbit(a, l), gb = stm_gbit(b, l);
          const unsigned long long xa = stm_rbit(a), xb = stm_rbit(b);
          const unsigned long long g1 = gc[k1][h] - ga + gb, g2 = gc[k2][h] - gb + ga;
          const unsigned long long r1 = rc[k1][h] - xa + xb, r2 = rc[k2][h] - xb + xa;
          const int before = stm_nib_max(gc[k1][h]) + stm_nib_max(gc[k2][h]) +
                             2 * (stm_nib_max(rc[k1][h]) + stm_nib_max(rc[k2][h]));
          const int after = stm_nib_max(g1) + stm_nib_max(g2) + 2 * (stm_nib_max(r1) + stm_nib_max(r2));
          if (after >= before) continue;
          any = true;
          g[k1 * 32 + l] = b;
          g[k2 * 32 + l] = a;
          gc[k1][h] = g1; gc[k2][h] = g2; rc[k1][h] = r1; rc[k2][h] = r2;
          if (a >> 31) { rows[k1][ra >> 6] &= ~(1ull << (ra & 63)); rows[k2][ra >> 6] |= 1ull << (ra & 63); }
          if (b >> 31) { rows[k2][rb >> 6] &= ~(1ull << (rb & 63)); rows[k1][rb >> 6] |= 1ull << (rb & 63); }
        }
    }
    if (!any) break;
  }
  for (int i = 0; i < D * 32; ++i) {
    const unsigned c = g[i];
    if (!(c >> 31)) continue;
    const long long e = p0 + (c & 2047u);
    slot[e] = (slot[e] & (1 << 30)) | i;
  }
}

__global__ void k_stm_pin(const long long* sec_ptr, long long nsec, unsigned long long* key,
                          int* perm, int* slot, unsigned short* depth, unsigned char* hown) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long s = tid; s < nsec; s += nt) {
    const long long p0 = sec_ptr[s], p1 = sec_ptr[s + 1];
    const long long E = p1 - p0;
    for (int l = 0; l < 32; ++l) hown[s * 32 + l] = 0xff;
    if (E == 0) { depth[s] = 0; continue; }
    const int D0 = (int)((E + 31) / 32);
    if (D0 > kStmPinMax) { depth[s] = 0xffff; continue; }
    int cnt[32], host[32];
    long long run0[32];
    unsigned freem[kStmPinMax];
    int ostep[kStmPinMax];
    for (int l = 0; l < 32; ++l) cnt[l] = 0;
    for (long long e = p0; e < p1; ++e) cnt[(key[e] >> 7) & 31u]++;
    {
      long long r = p0;
      for (int l = 0; l < 32; ++l) { run0[l] = r; r += cnt[l]; }
    }
    bool ok = false;
    int D = D0;
    for (; !ok && D <= 2 * D0 + 16 && D <= kStmPinMax; ++D) {
      // lanes that are not full start their pinned entries at step
      // rot(l) = l mod D (wrapping), so the free slots spread over all steps
      for (int k = 0; k < D; ++k) {
        unsigned m = 0;
        for (int l = 0; l < 32; ++l) {
          const int r = cnt[l] >= D ? 0 : l % D;
          m |= (((k - r + D) % D) >= cnt[l] ? 1u : 0u) << l;
        }
        freem[k] = m;
      }
      ok = true;
      unsigned done = 0;
      for (int l = 0; l < 32; ++l) host[l] = -1;  // a lane hosts the overflow of one owner
      for (int g = 0; g < 32 && ok; ++g) {  // owners by overflow size, descending
        int l = -1, o = 0;
        for (int c = 0; c < 32; ++c)
          if (!(done >> c & 1u) && cnt[c] - D > o) { o = cnt[c] - D; l = c; }
        if (l < 0) break;
        done |= 1u << l;
        // steps where the partner lane l ^ 16 (same accumulator banks as l,
        // other half-warp) is free first: hosting there adds no bank conflict
        unsigned allow = 0;
        for (int c = 0; c < 32; ++c)
          if (c != l && (host[c] < 0 || host[c] == l)) allow |= 1u << c;
        const unsigned partner = (1u << (l ^ 16)) & allow;
        int n = 0;
        for (int k = D - 1; k >= 0 && n < o; --k)
          if (freem[k] & partner) ostep[n++] = k;
        for (int k = D - 1; k >= 0 && n < o; --k)
          if ((freem[k] & allow) && !(freem[k] & partner)) ostep[n++] = k;
        if (n < o) { ok = false; break; }
        const long long run = run0[l];
        for (int q = 0; q < o && ok; ++q) {  // row-distinct steps: swap pinned entries
          const long long a = run + ostep[q], b = run + D + q;
          const unsigned jb = (unsigned)(key[b] & 7u);
          if ((unsigned)(key[a] & 7u) != jb) continue;
          bool fixed = false;
          for (int k2 = 0; k2 < D && !fixed; ++k2) {
            const long long c2 = run + k2;
            if ((unsigned)(key[c2] & 7u) == jb) continue;
            int q2 = -1;  // overflow entry of this owner at step k2, if any
            for (int t = 0; t < o; ++t)
              if (ostep[t] == k2) q2 = t;
            if (q2 >= 0 && (unsigned)(key[run + D + q2] & 7u) == jb) continue;
            const unsigned long long tk = key[a]; key[a] = key[c2]; key[c2] = tk;
            const int tp = perm[a]; perm[a] = perm[c2]; perm[c2] = tp;
            fixed = true;
          }
          ok = fixed;
        }
        for (int q = 0; q < o && ok; ++q) {
          const int k = ostep[q];
          const unsigned m = freem[k] & allow;
          int lane = -1;  // prefer the partner, then a lane already hosting l
          if (m & partner) lane = l ^ 16;
          for (int c = 0; c < 32 && lane < 0; ++c)
            if ((m >> c & 1u) && host[c] == l) lane = c;
          if (lane < 0) lane = __ffs(m) - 1;
          host[lane] = l;
          freem[k] &= ~(1u << lane);
          slot[run + D + q] = (k * 32 + lane) | (1 << 30);
        }
      }
      if (ok) {
        // gather banks of a step, per half-warp (the shared-memory conflict
        // unit of 8-byte loads): first the entries whose step is fixed
        // (owner lanes' pinned entries, overflow entries), then every other
        // lane picks, step by step, the remaining entry of its run whose
        // bank is least used at that step in its half-warp
        // (16-byte gathers of NV = 2 passes conflict per quarter-warp over
        // 8 bank quads: those counts weigh 4x in the choice)
        unsigned char use[kStmPinMax][2][16], useq[kStmPinMax][4][8];
        for (int k = 0; k < D; ++k) {
          for (int h = 0; h < 2; ++h)
            for (int b = 0; b < 16; ++b) use[k][h][b] = 0;
          for (int h = 0; h < 4; ++h)
            for (int b = 0; b < 8; ++b) useq[k][h][b] = 0;
        }
        auto bank = [&](long long e) {
          return (unsigned)(((key[e] >> 3) + (key[e] >> 7)) & 15u);  // (col - lane) + lane
        };
        for (int l = 0; l < 32; ++l) {
          if (cnt[l] <= D) continue;
          for (int i = 0; i < D; ++i) {
            const long long e = run0[l] + i;
            slot[e] = i * 32 + l;
            use[i][l >> 4][bank(e)]++;
            useq[i][l >> 3][bank(e) & 7u]++;
          }
          for (long long e = run0[l] + D; e < run0[l] + cnt[l]; ++e) {
            const int sl = slot[e] & ((1 << 30) - 1);
            use[sl >> 5][(sl & 31) >> 4][bank(e)]++;
            useq[sl >> 5][(sl & 31) >> 3][bank(e) & 7u]++;
          }
        }
        for (int l = 0; l < 32; ++l) {
          if (cnt[l] > D) continue;
          const int r = cnt[l] >= D ? 0 : l % D;
          for (int i = 0; i < cnt[l]; ++i) {
            const int k = (i + r) % D;
            long long best = run0[l] + i;
            int bu = 1 << 30;
            // candidates: the next 8 entries of the run (keeps deep sections linear)
            const long long e_end = run0[l] + (cnt[l] < i + 8 ? cnt[l] : i + 8);
            for (long long e = run0[l] + i; e < e_end; ++e) {
              const unsigned b = bank(e);
              const int u = 4 * useq[k][l >> 3][b & 7u] + use[k][l >> 4][b];
              if (u < bu) { bu = u; best = e; }
            }
            const long long a = run0[l] + i;
            if (best != a) {
              const unsigned long long tk = key[a]; key[a] = key[best]; key[best] = tk;
              const int tp = perm[a]; perm[a] = perm[best]; perm[best] = tp;
            }
            use[k][l >> 4][bank(a)]++;
            useq[k][l >> 3][bank(a) & 7u]++;
            slot[a] = k * 32 + l;
          }
        }
        if (D <= kStmSearchMax && E <= 2047) stm_search(key, p0, E, D, slot);
      }
    }
    if (!ok) { depth[s] = 0xffff; continue; }
    for (int l = 0; l < 32; ++l) hown[s * 32 + l] = host[l] < 0 ? 0xff : (unsigned char)host[l];
    depth[s] = (unsigned short)(D - 1);  // the loop stepped past the depth that worked
  }
}

// piece headers, owner tables, padding (values 0, padding words): one warp
// per piece
__global__ void k_stm_init(unsigned char* blob, const unsigned long long* poff, const unsigned* pslots,
                           const unsigned short* pwsec, const long long* ptile,
                           const unsigned char* hown, long long npiece) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long p = w; p < npiece; p += nw) {
    unsigned char* b = blob + poff[p];
    const unsigned ns = pslots[p];
    if (lane == 0) *reinterpret_cast<unsigned*>(b) = ns;
    if (lane < kStmWarps + 1)
      reinterpret_cast<unsigned short*>(b + 4)[lane] = pwsec[p * (kStmWarps + 1) + lane];
    const long long sec0 = ptile[p] * kStmWarps;
    for (int q = lane; q < kStmWarps * 32; q += 32) b[kStmHdr + q] = hown[sec0 * 32 + q];
    double* v = reinterpret_cast<double*>(b + kStmData);
    unsigned short* id = reinterpret_cast<unsigned short*>(b + kStmData + 8 * (size_t)ns);
    // padding gathers column = lane: distinct banks, no conflict with the real entries
    for (unsigned k = lane; k < ns; k += 32) {
      v[k] = 0.0;
      id[k] = (unsigned short)lane;
    }
  }
}

// scatter every entry of a tiled sub-block into its piece
__global__ void k_stm_scatter(const int* sec, const int* slot, long long nnz, const int* perm,
                              const int* rowid, const int* ci, const double* val,
                              const long long* tile_pf, const unsigned short* pstep0,
                              const int* tile_np,
                              const unsigned long long* poff, const unsigned* pslots,
                              const unsigned short* pwsec, int W, unsigned char* blob) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long e = tid; e < nnz; e += nt) {
    const int sc = sec[e];
    const long long tile = sc / kStmWarps;
    const int w = sc % kStmWarps;
    const long long pf = tile_pf[tile];
    if (pf < 0) continue;  // CSR sub-block
    const int sl = slot[e];
    const unsigned ovf = (unsigned)(sl >> 30) & 1u;
    const int k = (sl & ((1 << 30) - 1)) >> 5, lane = sl & 31;
    long long piece = pf;  // the piece whose step range holds step k
    for (const long long pend = pf + tile_np[tile]; piece + 1 < pend && pstep0[piece + 1] <= k;) ++piece;
    const int kk = k - pstep0[piece];
    unsigned char* bl = blob + poff[piece];
    const unsigned ns = pslots[piece];
    const long long at = ((long long)pwsec[piece * (kStmWarps + 1) + w] + kk) * 32 + lane;
    const int s = perm[e];
    const unsigned rl = (unsigned)(rowid[s] % kStmSecRows);
    reinterpret_cast<double*>(bl + kStmData)[at] = val[s];
    reinterpret_cast<unsigned short*>(bl + kStmData + 8 * (size_t)ns)[at] =
        (unsigned short)((unsigned)(ci[s] % W) | ((rl >> 5) << 12) | (ovf << 15));
  }
}

}  // namespace scs
