// kernels.cuh -- the per-iteration device kernels of the indirect SCS path.
//
// One ADMM iteration (solver.py:153-166 + 355-363) is this fixed kernel
// sequence, captured once into a CUDA graph; every data-dependent branch of
// the reference (CG early exits, termination) is taken on the device from
// the Ctl block, so the host never synchronises inside an iteration:
//
//   k_prep         w = u+v, rhs = w[:-1] - w_tau h, ||rhs|| -> CG tol       embedding.py:177-185
//   SpMV A^T  [EpiAtFirst]  cg_rhs = rhs_x - A^T rhs_y, r0 = cg_rhs - G x0   embedding.py:109, sparse_linalg.py:264-272
//                           (+ A^T u_y of the previous iterate, see below --
//                           every R-th iteration; the others run EpiAtFirst1,
//                           NV = 1, with A^T u_y from recurrences)
//   cg_max x { SpMV A [EpiAp]; SpMV A^T [EpiAtGp]; k_cg_update; k_cg_p }    sparse_linalg.py:273-288
//                           (the first A pass also carries A u_x, below --
//                           every R-th iteration; the others carry A u_x by
//                           recurrence in k_cone_tail, SCS_RES_RECUR)
//   SpMV A    [EpiAFinal]   z_y = rhs_y + A x, corr = h'p / denom          embedding.py:113, 192
//   k_cone_tail    u~, relaxation, cone projection (elementwise / SOC / exp),
//                  tau update                                               embedding.py:193-196, solver.py:163-165
//   k_cone_apply   large SOC + PSD (Jacobi) blocks                          cones.py:172-191
//
// Matrix passes per iteration: 2 + 2k (k = CG steps); the reference makes 6 + 2k
// (k = CG steps, sparse_linalg.py:264,471,486 + embedding.py:109,113 +
// scaling.py:165-166).  Removed, with bit-identical results:
//  * A x_warm at the head of CG: the previous iteration's EpiAFinal already
//    produced A x for the same x (cg_warm) and stored it (Axw);
//  * the trailing exact-residual pass (sparse_linalg.py:289), whose value
//    its caller discards (embedding.py:110);
//  * the two residual passes of the termination check (scaling.py:165-166):
//    they gather the same interleaved sector as the next iteration's first
//    A^T / A pass, so they ride along; the next iteration is speculative
//    until the check of the previous one has passed (its state writes come
//    after the check), exactly reproducing the reference's loop exit.
#pragma once

#include "common.cuh"
#include "cones.cuh"

namespace scs {

struct Csr {
  const long long* rp;  // rows + 1
  const int* ci;        // nnz
  const double* v;      // nnz
  long long rows;
};

// Device vectors of one handle.  x-part length n, y-part length m (local).
// Gather vectors are interleaved so that one 16-byte load (one sector
// request) serves every SpMV that shares a matrix pass:
//   X2[2j + 0] = p_j (CG direction)          X2[2j + 1] = (u_x)_j
//   Y2[2i + 0] = (rhs_y + A cg_warm)_i       Y2[2i + 1] = (u_y)_i
// The first A^T pass forms A^T rhs_y + A^T (A x0) as A^T (rhs_y + A x0):
// same products, one gather (a rounding-level reassociation).
struct Vec {
  long long n, m;
  double *u, *v;              // n + m + 1 (SolverState)
  const double *c, *b;        // scaled data
  const double *D, *E;        // scalings
  const double *Dinv, *Einv;  // 1/D, 1/E (scaling.py:163-164)
  double *gx, *gy;            // g = M^-1 h
  double *rhs_x, *rhs_y;      // rhs = w[:-1] - w_tau h
  double *x;                  // CG iterate == cg_warm (embedding.py:111)
  const double* Minv;         // opt-in Jacobi PCG: 1 / diag(I + A^T A); nullptr = plain CG
  double *r, *Gp;             // CG vectors (n)
  double *X2, *Y2;            // interleaved gather vectors
  double *P1;                 // compact copy of p = X2[2j] (stride-1 gathers of the later CG A passes)
  double *Axw;                // A cg_warm (m), from the previous EpiAFinal
  double *Aux;                // A u_x (m) for the split residual epilogue
  double *Agx;                // A g_x (m): residual recurrence on (nullptr: off)
  // A^T side of the residual recurrence (n each; T == nullptr: off):
  double *T;                  // A^T A x of the CG iterate (carried through the Gp products)
  double *AtAp;               // A^T A p of the current CG step (EpiAtGp), for T
  double *Sv;                 // A^T rhs_y of this iteration
  double *Uy;                 // A^T u_y of the current state
  double *Dd;                 // A^T (v_y - u_y) of the current state
  double *Atb, *Atgy;         // A^T b^, A^T g_y (setup)
  double *Yc;                 // compact rhs_y + A cg_warm (m), gather of the NV = 1 first pass
  double *q;                  // A p (m)
  double *zy;                 // z_y = rhs_y + A x (m)
  double *part;               // kMaxRed * kMaxGrid partials
  double *dred;               // deferred (to-be-all-reduced) totals, kMaxRed
  double xw;                  // weight of replicated x-part terms in
                              // all-reduced sums: 1 on rank 0, else 0
  double *chunk_part;         // big-SOC chunk partial norms
  double *soc_fac;            // 3 per big SOC: mode, head, scale
  double *cone_red;           // [c'u~x, b'u~y, err, then (||z||^2, t0) per global big SOC]
  double *dbg;                // SCS_DEBUG_PSD: first non-converged PSD block (flag, side, svec)
  Ctl* ctl;
};

// Cone layout of the local y-part (cones.py:121-139 order + exp last).
struct Cones {
  long long z, l;                 // [0, z) zero, [z, z + l) nonneg
  int n_ssoc;                     // small SOCs (<= kSmallSoc): warp per cone
  const long long* ssoc_off;      // start of each small SOC
  const int* ssoc_len;            // its dimension
  int n_bsoc;                     // big SOCs: chunked
  const long long* bsoc_off;      // n_bsoc start offsets
  const long long* bsoc_len;
  const int* bsoc_chunk_lo;       // n_bsoc + 1
  int n_chunk;
  const long long* chunk_off;     // chunk start (absolute y offset)
  const int* chunk_len;
  const int* chunk_cone;
  const int* bsoc_gid;            // global id of each big SOC (all-reduce slot)
  int n_big_global;               // big-path SOCs over all shards
  int n_psd;
  const long long* psd_off;
  const int* psd_side;
  const long long* psd_goff;      // global scratch offset of blocks beyond the smem side (-1: smem)
  long long psd_lo, psd_hi;       // y range of all PSD blocks
  long long exp_lo;               // first exp row
  long long n_exp;
  int max_side;
};

constexpr int kSmallSoc = 2048;  // warp-per-cone bound
constexpr int kChunk = 1024;     // big-SOC chunk (one CTA)

// ---------------------------------------------------------------------------
// CSR row dot products: L lanes per row, lane-strided, FMA, group shuffle.
// The matrix streams (ci, v) are loaded with evict-first (ld.global.cs) so
// the L2 keeps the gather vectors resident.  NV values are gathered per
// nonzero from an interleaved vector (STRIDE doubles per entry) with one
// load instruction: 64-bit, 128-bit (double2) or 256-bit (v4.f64).
// ---------------------------------------------------------------------------
template <int NV, int STRIDE>
__device__ __forceinline__ void gather(const double* __restrict__ xb, int c, double (&g)[NV]) {
  const double* p = xb + (size_t)c * STRIDE;
  if constexpr (NV == 1) {
    g[0] = __ldg(p);
  } else if constexpr (NV == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    g[0] = t.x;
    g[1] = t.y;
  } else {
    static_assert(STRIDE == 4 && NV <= 4, "256-bit gathers need a stride of 4");
    double a, b, cc, d;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(cc), "=d"(d) : "l"(p));
    g[0] = a;
    g[1] = b;
    if constexpr (NV > 2) g[2] = cc;
    if constexpr (NV > 3) g[3] = d;
  }
}

template <int L, int NV, int STRIDE>
__device__ __forceinline__ void row_dot(const Csr& A, long long k0, long long k1, int gl,
                                        const double* __restrict__ xb, double (&s)[NV]) {
#pragma unroll
  for (int t = 0; t < NV; ++t) s[t] = 0.0;
  // every step issues up to four predicated (column, value) loads per lane
  // before any gather, so short rows keep as many loads in flight as long ones
  for (long long k = k0 + gl; k < k1; k += 4 * L) {
    int c[4];
    double a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = k + u * L < k1;
      c[u] = ok ? __ldcs(A.ci + k + u * L) : 0;
      a[u] = ok ? __ldcs(A.v + k + u * L) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (k + u * L < k1) {
        double g[NV];
        gather<NV, STRIDE>(xb, c[u], g);
#pragma unroll
        for (int t = 0; t < NV; ++t) s[t] = fma(a[u], g[t], s[t]);
      }
    }
  }
  // all 32 lanes reach the shuffles: the row loop below is warp-uniform
#pragma unroll
  for (int t = 0; t < NV; ++t) s[t] = group_sum<L>(s[t]);
}

// Generic CSR SpMV with a per-row epilogue and an optional grid reduction
// whose last block runs Epi::finish.  Each warp owns 32/L consecutive rows
// per step (L lanes per row); the row loop is warp-uniform so the group
// shuffles never see diverged lanes.  The next row's pointers are fetched
// one step ahead and the epilogue operands before the dot product, so the
// matrix stream is the only dependent latency per row.  Epi::load() reads
// the Ctl flags once and says whether the whole launch is a no-op.
template <int L, class Epi>
__global__ void __launch_bounds__(kBlock, Epi::MINB) k_spmv(Csr A, Epi epi0) {
  Epi epi = epi0;
  if (!epi.load()) return;
  constexpr int kGroups = 32 / L;
  constexpr int NR = Epi::NR > 0 ? Epi::NR : 1;
  const int gl = threadIdx.x & (L - 1);
  const int gi = (threadIdx.x & 31) / L;
  const long long warp = ((long long)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * kBlock) >> 5;
  const long long stride = nwarps * kGroups;
  double red[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) red[t] = 0.0;
  long long base = warp * kGroups;
  long long row = base + gi;
  bool valid = row < A.rows;
  long long k0 = 0, k1 = 0;
  if (valid) { k0 = __ldg(A.rp + row); k1 = __ldg(A.rp + row + 1); }
  for (; base < A.rows; base += stride) {
    const long long nrow = row + stride;
    const bool nvalid = nrow < A.rows;
    long long nk0 = 0, nk1 = 0;
    if (nvalid) { nk0 = __ldg(A.rp + nrow); nk1 = __ldg(A.rp + nrow + 1); }
    typename Epi::Pre pre;
    if (valid) epi.pre(row, pre);
    double s[Epi::NV];
    row_dot<L, Epi::NV, Epi::STRIDE>(A, k0, k1, gl, epi.xb, s);
    if (valid && gl == 0) epi.row(row, s, pre, red);
    row = nrow;
    valid = nvalid;
    k0 = nk0;
    k1 = nk1;
  }
  epi.extra(red);
  if constexpr (Epi::NR > 0) {
    if (grid_sum_last<Epi::NR>(red, epi.V.part, &epi.V.ctl->counter)) {
      if (epi.defer) {  // row-sharded: totals are all-reduced, then k_finish
        if (threadIdx.x == 0)
          for (int t = 0; t < Epi::NR; ++t) epi.V.dred[t] = red[t];
      } else {
        epi.finish(red);
      }
    }
  }
}

// Row-sharded A^T pass, part 1: raw partial products T[j*NV + t] of the
// local rows of A (= local columns of A^T); all-reduced before part 2.
template <class Inner>
struct EpiRaw : Inner {
  static constexpr int NR = 0;
  double* T;
  struct Pre {};
  __device__ void pre(long long, Pre&) const {}
  __device__ void row(long long j, const double (&s)[Inner::NV], const Pre&, double*) const {
#pragma unroll
    for (int t = 0; t < Inner::NV; ++t) T[j * Inner::NV + t] = s[t];
  }
  __device__ void extra(double*) const {}
  __device__ void finish(const double*) const {}
};

// Split long rows with more than kLongSeg pieces: in k_rows, one warp per
// such row sums its pieces (lane-strided, then a butterfly: a fixed order)
// and its lane 0 runs the row's epilogue (r01: a separate k_seg_long launch
// wrote the sums back for k_rows -- 11 us of config 4's 41-us A pass).
constexpr int kLongSeg = 32;

// Row-sharded or row-banded A^T pass, part 2: the epilogue over the
// all-reduced products, or over the sum of `nsum` band partials (in band
// order; stride rows * NV), or -- split long rows, `seg` != nullptr -- over
// the sum of row i's pieces seg[i] .. seg[i+1]-1 (in order).
template <class Epi>
__global__ void __launch_bounds__(kBlock) k_rows(const double* T, long long rows, int nsum, Epi epi0,
                                                 const long long* seg = nullptr,
                                                 const long long* long_rows = nullptr,
                                                 long long n_long = 0) {
  Epi epi = epi0;
  if (!epi.load()) return;
  constexpr int NR = Epi::NR > 0 ? Epi::NR : 1;
  double red[NR];
#pragma unroll
  for (int t = 0; t < NR; ++t) red[t] = 0.0;
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  if (seg && n_long) {  // long rows: a warp each
    const int lane = threadIdx.x & 31;
    for (long long r = tid >> 5; r < n_long; r += nt >> 5) {
      const long long j = long_rows[r], v0 = seg[j], v1 = seg[j + 1];
      double s[Epi::NV];
#pragma unroll
      for (int t = 0; t < Epi::NV; ++t) s[t] = 0.0;
      for (long long v = v0 + lane; v < v1; v += 32)
#pragma unroll
        for (int t = 0; t < Epi::NV; ++t) s[t] += T[v * Epi::NV + t];
#pragma unroll
      for (int t = 0; t < Epi::NV; ++t) s[t] = warp_sum(s[t]);
      if (lane == 0) {
        typename Epi::Pre pre;
        epi.pre(j, pre);
        epi.row(j, s, pre, red);
      }
    }
  }
  for (long long j = tid; j < rows; j += nt) {
    long long v0 = 0, v1 = 0;
    if (seg) {
      v0 = seg[j];
      v1 = seg[j + 1];
      if (v1 - v0 > kLongSeg) continue;  // a warp's (above)
    }
    typename Epi::Pre pre;
    epi.pre(j, pre);
    double s[Epi::NV];
    if (seg) {
#pragma unroll
      for (int t = 0; t < Epi::NV; ++t) s[t] = T[v0 * Epi::NV + t];
      for (long long v = v0 + 1; v < v1; ++v)
#pragma unroll
        for (int t = 0; t < Epi::NV; ++t) s[t] += T[v * Epi::NV + t];
    } else {
#pragma unroll
      for (int t = 0; t < Epi::NV; ++t) s[t] = T[j * Epi::NV + t];
      int b = 1;
      for (; b + 4 <= nsum; b += 4) {  // four partials' loads in flight, added in order
        double v[4][Epi::NV];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int t = 0; t < Epi::NV; ++t) v[q][t] = T[((b + q) * rows + j) * Epi::NV + t];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int t = 0; t < Epi::NV; ++t) s[t] += v[q][t];
      }
      for (; b < nsum; ++b)
#pragma unroll
        for (int t = 0; t < Epi::NV; ++t) s[t] += T[(b * rows + j) * Epi::NV + t];
    }
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

// Deferred finish after the all-reduce of V.dred (one block).
template <class Epi>
__global__ void k_finish(Epi epi0) {
  Epi epi = epi0;
  if (!epi.load()) return;
  double tot[Epi::NR > 0 ? Epi::NR : 1];
  for (int t = 0; t < Epi::NR; ++t) tot[t] = epi.V.dred[t];
  epi.finish(tot);
}

__device__ void finish_residuals(Ctl* c, double ut, double s_pri, double s_unb, double buy,
                                 double s_dual, double s_inf, double cux);

// ---- epilogues --------------------------------------------------------------
struct EpiBase {
  Vec V;
  const double* xb;  // gather base
  int pend;          // residual check of the previous iteration rides along
  int defer;         // row-sharded: totals go to V.dred for an all-reduce
  // residual recurrence (first CG pass): +R = run on refresh iterations
  // (k_sched = 1, 1 + R, ...), -R = run on the others, 0 = always
  int rgate;
  int waux;          // refresh pass: always store A u_x into Aux
  static constexpr int MINB = 1;  // min resident CTAs per SM (register cap)
  __device__ __forceinline__ bool gate_ok() const {
    if (!rgate) return true;
    const int R = rgate > 0 ? rgate : -rgate;
    const bool refresh = (V.ctl->k_sched - 1) % R == 0;
    return refresh == (rgate > 0);
  }
  struct Pre {};
  __device__ void pre(long long, Pre&) const {}
  __device__ void extra(double*) const {}
  __device__ __forceinline__ double utau() const { return V.u[V.n + V.m]; }
};

// First A^T pass of an iteration (sparse_linalg.py:264-272 + scaling.py:166):
//   r0 = (rhs_x - x0) - A^T (rhs_y + A x0); p = r0
// and, when the previous iteration is due a termination check, A^T u_y of
// that iterate (dual residual / infeasibility, scaling.py:183-189).  One
// 128-bit gather per nonzero serves both products.
struct EpiAtFirst : EpiBase {
  static constexpr int NV = 2, STRIDE = 2, NR = 5;
  __device__ bool load() {
    pend = V.ctl->check_pending;
    return gate_ok() && !V.ctl->stop;
  }
  struct Pre { double rx, x, mi, ei, c, ux, ut; };
  __device__ void pre(long long j, Pre& p) const {
    p.rx = V.rhs_x[j];
    p.x = V.x[j];
    if (V.Minv) p.mi = V.Minv[j];
    if (pend) { p.ei = V.Einv[j]; p.c = V.c[j]; p.ux = V.X2[2 * j + 1]; p.ut = utau(); }
  }
  __device__ void row(long long j, const double (&s)[2], const Pre& p, double* red) const {
    const double r = (p.rx - p.x) - s[0];
    V.r[j] = r;
    red[0] += r * r;
    if (V.Minv) {  // opt-in PCG: p = z = M^-1 r, carry r'z
      const double z = p.mi * r;
      V.X2[2 * j] = z;
      V.P1[j] = z;
      red[4] += r * z;
    } else {
      V.X2[2 * j] = r;
      V.P1[j] = r;
    }
    if (pend) {
      const double du = p.ei * (s[1] / p.ut + p.c);
      const double inf = p.ei * s[1];
      red[1] += du * du;
      red[2] += inf * inf;
      red[3] += p.c * p.ux;
    }
    if (rgate > 0) {  // refresh of the A^T-side recurrence (T just computed directly)
      const double sv = s[0] - V.T[j];
      V.Sv[j] = sv;
      V.Uy[j] = s[1];
      V.Dd[j] = (sv + (V.u[V.n + V.m] + V.v[V.n + V.m]) * V.Atb[j]) - 2.0 * s[1];
    }
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    Ctl* c = V.ctl;
    if (pend) { c->sums[3] = tot[1]; c->sums[4] = tot[2]; c->sums[5] = tot[3]; }
    const double res = sqrt(tot[0]);
    c->cg_it = 0;
    if (!isfinite(res)) { c->err |= ERR_CG_NONFINITE; c->stop = 1; c->cg_done = 1; return; }
    if (res <= c->tol) { c->cg_done = 1; return; }
    c->cg_done = 0;
    c->rs = V.Minv ? tot[4] : res * res;
  }
};

// First A^T pass with the A^T-side residual recurrence (non-refresh
// iterations): one product F = A^T (rhs_y + A x0) from the compact gather Yc.
// With T = A^T A x0 carried by the CG updates, A^T rhs_y = F - T, and since
// rhs_y = u_y + v_y - w_tau b^ (embedding.py:177-178),
//   A^T u_y = ((F - T) + w_tau A^T b^ - Dd) / 2,   Dd = A^T (v_y - u_y)
// (Dd from k_cone_tail: v+ - u+ = v - u_bar, solver.py:165).
struct EpiAtFirst1 : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 5;
  __device__ bool load() {
    pend = V.ctl->check_pending;
    return gate_ok() && !V.ctl->stop;
  }
  struct Pre { double rx, x, mi, ei, c, ux, ut, wt; };
  __device__ void pre(long long j, Pre& p) const {
    p.rx = V.rhs_x[j];
    p.x = V.x[j];
    if (V.Minv) p.mi = V.Minv[j];
    p.ut = utau();
    p.wt = p.ut + V.v[V.n + V.m];
    if (pend) { p.ei = V.Einv[j]; p.c = V.c[j]; p.ux = V.X2[2 * j + 1]; }
  }
  __device__ void row(long long j, const double (&s)[1], const Pre& p, double* red) const {
    const double r = (p.rx - p.x) - s[0];
    V.r[j] = r;
    red[0] += r * r;
    if (V.Minv) {
      const double z = p.mi * r;
      V.X2[2 * j] = z;
      V.P1[j] = z;
      red[4] += r * z;
    } else {
      V.X2[2 * j] = r;
      V.P1[j] = r;
    }
    const double sv = s[0] - V.T[j];
    const double uy = 0.5 * ((sv + p.wt * V.Atb[j]) - V.Dd[j]);
    V.Sv[j] = sv;
    V.Uy[j] = uy;
    if (pend) {
      const double du = p.ei * (uy / p.ut + p.c);
      const double inf = p.ei * uy;
      red[1] += du * du;
      red[2] += inf * inf;
      red[3] += p.c * p.ux;
    }
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    Ctl* c = V.ctl;
    if (pend) { c->sums[3] = tot[1]; c->sums[4] = tot[2]; c->sums[5] = tot[3]; }
    const double res = sqrt(tot[0]);
    c->cg_it = 0;
    if (!isfinite(res)) { c->err |= ERR_CG_NONFINITE; c->stop = 1; c->cg_done = 1; return; }
    if (res <= c->tol) { c->cg_done = 1; return; }
    c->cg_done = 0;
    c->rs = V.Minv ? tot[4] : res * res;
  }
};

// EpiAtFirst1, split (one GPU, no bands): the pass only stores F into Sv,
// then k_rows runs EpiAtFirst1 over it (a heavy per-row epilogue inside the
// streamed kernel cost ~0.55 ms at config 5; coalesced, it is ~20 us).
struct EpiStoreF : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 0;
  __device__ bool load() { return gate_ok() && !V.ctl->stop; }
  __device__ void row(long long j, const double (&s)[1], const Pre&, double*) const { V.Sv[j] = s[0]; }
  __device__ void finish(const double*) const {}
};

// Refresh of T = A^T (A x0) (A x0 = Axw, stored by the previous final pass).
struct EpiTRef : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 0;
  __device__ bool load() { return gate_ok() && !V.ctl->stop; }
  __device__ void row(long long j, const double (&s)[1], const Pre&, double*) const { V.T[j] = s[0]; }
  __device__ void finish(const double*) const {}
};

// q = A p.  MERGED: the first CG pass also carries A u_x of the previous
// iterate (primal residual / unboundedness, scaling.py:165-188) and closes
// that iteration's termination check (solver.py:359-363).
template <bool MERGED>
struct EpiAp : EpiBase {
  // MERGED gathers [p, u_x] from X2; plain passes gather p from its compact copy P1
  static constexpr int NV = MERGED ? 2 : 1, STRIDE = MERGED ? 2 : 1, NR = MERGED ? 3 : 0;
  __device__ bool load() {
    const Ctl* c = V.ctl;
    pend = MERGED ? c->check_pending : 0;
    if (!gate_ok()) return false;
    return !c->stop && (!c->cg_done || pend || waux);
  }
  struct Pre { double vs, d, b, uy, ut; };
  __device__ void pre(long long i, Pre& p) const {
    if constexpr (MERGED) {
      if (pend) {
        p.vs = V.v[V.n + i]; p.d = V.Dinv[i]; p.b = V.b[i]; p.uy = V.Y2[2 * i + 1]; p.ut = utau();
      }
    }
  }
  __device__ void row(long long i, const double (&s)[NV], const Pre& p, double* red) const {
    V.q[i] = s[0];
    if constexpr (MERGED) {
      if (waux) V.Aux[i] = s[1];
      if (pend) {
        const double t = s[1] + p.vs;
        const double di = p.d;
        const double pr = di * (t / p.ut - p.b);
        const double ub = di * t;
        red[0] += pr * pr;
        red[1] += ub * ub;
        red[2] += p.b * p.uy;
      }
    }
  }
  __device__ void finish(const double* tot) const {
    if constexpr (MERGED) {
      if (threadIdx.x || !pend) return;
      Ctl* c = V.ctl;
      finish_residuals(c, utau(), tot[0], tot[1], tot[2], c->sums[3], c->sums[4], c->sums[5]);
      c->check_pending = 0;
      if (c->stop) c->k_sched -= 1;  // the speculative iteration never happened
    }
  }
};

// Gp = p + A^T q, p'Gp -> alpha (sparse_linalg.py:274-278)
struct EpiAtGp : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 1;
  __device__ bool load() { return !V.ctl->stop && !V.ctl->cg_done; }
  struct Pre { double p; };
  __device__ void pre(long long j, Pre& p) const { p.p = V.X2[2 * j]; }
  __device__ void row(long long j, const double (&s)[1], const Pre& pf, double* red) const {
    const double pj = pf.p;
    const double g = pj + s[0];
    V.Gp[j] = g;
    if (V.AtAp) V.AtAp[j] = s[0];  // T += alpha A^T A p without the Gp - p cancellation
    red[0] += pj * g;
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    Ctl* c = V.ctl;
    const double den = tot[0];
    if (!isfinite(den) || den <= 0.0) { c->err |= ERR_CG_CURVATURE; c->stop = 1; c->cg_done = 1; return; }
    c->cg_alpha = c->rs / den;
  }
};

// z_y = rhs_y + A x; store A x for the next warm start; h'p -> corr
// (embedding.py:113, 192).  In setup mode (g = M^-1 h) writes g_y and the
// Schur denominator instead (embedding.py:152-161).
struct EpiAFinal : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 2;
  double* zy_out;
  int setup;
  __device__ bool load() { return !V.ctl->stop; }
  struct Pre { double ry, b; };
  __device__ void pre(long long i, Pre& p) const { p.ry = V.rhs_y[i]; p.b = V.b[i]; }
  __device__ void row(long long i, const double (&s)[1], const Pre& p, double* red) const {
    const double z = p.ry + s[0];
    zy_out[i] = z;
    if (!setup) V.Axw[i] = s[0];
    red[1] += p.b * z;
  }
  __device__ void extra(double* red) const {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nt = (long long)gridDim.x * blockDim.x;
    for (long long j = tid; j < V.n; j += nt) red[0] += V.xw * (V.c[j] * V.x[j]);
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    Ctl* c = V.ctl;
    c->cg_iters_total += c->cg_it;
    const double hp = tot[0] + tot[1];
    if (setup) {
      c->denom = 1.0 + hp;
    } else {
      c->warm_zero = 0;
      c->corr = hp / c->denom;
    }
  }
};

// Stand-alone termination check (after the last iteration of a loop, or a
// forced residual evaluation): A u_x ...
struct EpiResA : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 3;
  double* store;  // A u_x of the checked state (V.Aux: reused by the extraction)
  __device__ bool load() {
    const Ctl* c = V.ctl;
    return !c->stop && (c->check_pending || c->force_check);
  }
  struct Pre { double vs, d, b, uy, ut; };
  __device__ void pre(long long i, Pre& p) const {
    p.vs = V.v[V.n + i]; p.d = V.Dinv[i]; p.b = V.b[i]; p.uy = V.u[V.n + i]; p.ut = utau();
  }
  __device__ void row(long long i, const double (&s)[1], const Pre& p, double* red) const {
    const double t = s[0] + p.vs;
    const double di = p.d;
    const double pr = di * (t / p.ut - p.b);
    const double ub = di * t;
    if (store) store[i] = s[0];
    red[0] += pr * pr;
    red[1] += ub * ub;
    red[2] += p.b * p.uy;
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    V.ctl->sums[0] = tot[0];
    V.ctl->sums[1] = tot[1];
    V.ctl->sums[2] = tot[2];
  }
};

// ... and A^T u_y, then the status (scaling.py:166-206, solver.py:210-234)
struct EpiResAt : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 3;
  double* store;  // A^T u_y of the checked state (V.Uy: reused by the extraction)
  __device__ bool load() {
    const Ctl* c = V.ctl;
    return !c->stop && (c->check_pending || c->force_check);
  }
  struct Pre { double e, c, ux, ut; };
  __device__ void pre(long long j, Pre& p) const {
    p.e = V.Einv[j]; p.c = V.c[j]; p.ux = V.u[j]; p.ut = utau();
  }
  __device__ void row(long long j, const double (&s)[1], const Pre& p, double* red) const {
    const double ei = p.e;
    const double du = ei * (s[0] / p.ut + p.c);
    const double inf = ei * s[0];
    red[0] += du * du;
    red[1] += inf * inf;
    red[2] += p.c * p.ux;
    if (store) store[j] = s[0];
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    Ctl* c = V.ctl;
    finish_residuals(c, utau(), c->sums[0], c->sums[1], c->sums[2], tot[0], tot[1], tot[2]);
    c->check_pending = 0;
  }
};

// ---- split epilogues (CSR path): the SpMV only stores its products, a
// coalesced elementwise pass (k_rows) does the per-row work.  On the CSR
// kernel a heavy per-row epilogue costs more than re-reading two m-vectors.

// merged first CG A pass, plain: q = A p and (check due) Aux = A u_x
struct EpiApPlain2 : EpiBase {
  static constexpr int NV = 2, STRIDE = 2, NR = 0;
  __device__ bool load() {
    const Ctl* c = V.ctl;
    pend = c->check_pending;
    if (!gate_ok()) return false;
    return !c->stop && (!c->cg_done || pend || waux);
  }
  __device__ void row(long long i, const double (&s)[2], const Pre&, double*) const {
    V.q[i] = s[0];
    if (pend || waux) V.Aux[i] = s[1];
  }
  __device__ void finish(const double*) const {}
};
// ... then the residual terms of A u_x and the termination check
// (scaling.py:165-188, solver.py:359-363): EpiAp<true>'s epilogue over Aux
struct EpiResY : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 3;
  __device__ bool load() {
    const Ctl* c = V.ctl;
    pend = c->check_pending;
    return gate_ok() && !c->stop && pend;
  }
  struct Pre { double vs, d, b, uy, ut; };
  __device__ void pre(long long i, Pre& p) const {
    p.vs = V.v[V.n + i]; p.d = V.Dinv[i]; p.b = V.b[i]; p.uy = V.Y2[2 * i + 1]; p.ut = utau();
  }
  __device__ void row(long long i, const double (&s)[1], const Pre& p, double* red) const {
    const double t = s[0] + p.vs;
    const double pr = p.d * (t / p.ut - p.b);
    const double ub = p.d * t;
    red[0] += pr * pr;
    red[1] += ub * ub;
    red[2] += p.b * p.uy;
  }
  __device__ void finish(const double* tot) const {
    if (threadIdx.x) return;
    Ctl* c = V.ctl;
    finish_residuals(c, utau(), tot[0], tot[1], tot[2], c->sums[3], c->sums[4], c->sums[5]);
    c->check_pending = 0;
    if (c->stop) c->k_sched -= 1;  // the speculative iteration never happened
  }
};
// final A pass, plain: Axw = A x.  Opt-in recurrence mode (gate > 0): A x
// is carried by k_cg_update (Axw += alpha q) and this pass only refreshes
// it directly every `gate` iterations (bounds the rounding drift).
struct EpiAxPlain : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 0;
  int gate;
  __device__ bool load() {
    const Ctl* c = V.ctl;
    return !c->stop && (gate <= 0 || c->k_sched % gate == 0);
  }
  __device__ void row(long long i, const double (&s)[1], const Pre&, double*) const { V.Axw[i] = s[0]; }
  __device__ void finish(const double*) const {}
};
// ... then z_y = rhs_y + A x and h'p (EpiAFinal's epilogue over Axw)
struct EpiZy : EpiAFinal {
  __device__ void row(long long i, const double (&s)[1], const Pre& p, double* red) const {
    const double z = p.ry + s[0];
    zy_out[i] = z;
    red[1] += p.b * z;
  }
};

// Plain products for the C-ABI test hook (scs_apply_a).
struct EpiPlain : EpiBase {
  static constexpr int NV = 1, STRIDE = 1, NR = 0;
  double* out;
  __device__ bool load() { return true; }
  __device__ void row(long long i, const double (&s)[1], const Pre&, double*) const { out[i] = s[0]; }
  __device__ void finish(const double*) const {}
};

// Plain two-vector products from an interleaved vector (format self-checks).
template <int NV_, int STRIDE_>
struct EpiPlainN : EpiBase {
  static constexpr int NV = NV_, STRIDE = STRIDE_, NR = 0;
  double* out;  // rows * NV
  __device__ bool load() { return true; }
  __device__ void row(long long i, const double (&s)[NV], const Pre&, double*) const {
#pragma unroll
    for (int t = 0; t < NV; ++t) out[i * NV + t] = s[t];
  }
  __device__ void finish(const double*) const {}
};

}  // namespace scs
