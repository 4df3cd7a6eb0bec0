// solver.cu -- B200-native SCS indirect-method hot path: device kernels that
// are not SpMV epilogues, the setup path (CSC ingest, device transpose,
// Ruiz equilibration, g = M^-1 h), the graph-captured iteration loop, and
// the C-ABI declared in include/scs_b200.h.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <errno.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include "../../include/scs_b200.h"
#include "common.cuh"
#include "cones.cuh"
#include "kernels.cuh"
#include "stream.cuh"

#ifdef SCS_WITH_NCCL
#include <nccl.h>
#endif

namespace scs {

// ===========================================================================
// iteration kernels (non-SpMV)
// ===========================================================================

// CG tolerance of this iteration from ||rhs||^2 (embedding.py:179-185)
__device__ void prep_finish(Ctl* c, double rhs2, int variant, int R) {
  const long long k = ++c->k_sched;
  // graph variant of this iteration (1: non-refresh, 2: refresh of the
  // residual recurrences, solver.cu run_iteration) must match the schedule
  // the gated epilogues use (kernels.cuh EpiBase::gate_ok)
  if (variant && ((k - 1) % R == 0) != (variant == 2)) { c->err |= ERR_SCHED; c->stop = 1; }
  c->tol = c->cg_tol > 0.0 ? c->cg_tol
                           : 1e-3 * (1.0 + sqrt(rhs2)) / pow((double)(k < 1 ? 1 : k), 1.5);
  c->cg_done = 0;
  c->cg_it = 0;
}

// w = u + v; rhs = w[:-1] - w_tau h; ||rhs||^2 (embedding.py:177-185).
// Row-sharded (defer): the x-part counts on rank 0 only (V.xw) and the
// total is all-reduced before k_prep_finish.
__global__ void __launch_bounds__(kBlock) k_prep(Vec V, int defer, int variant, int R) {
  Ctl* c = V.ctl;
  if (c->stop) return;
  const long long n = V.n, m = V.m;
  const double wt = V.u[n + m] + V.v[n + m];
  double red[1] = {0.0};
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  for (long long i = tid; i < n + m; i += nt) {
    const double w = V.u[i] + V.v[i];
    double r;
    if (i < n) {
      r = w - wt * V.c[i];
      V.rhs_x[i] = r;
      red[0] += V.xw * (r * r);
    } else {
      r = w - wt * V.b[i - n];
      V.rhs_y[i - n] = r;
      const double yv = r + V.Axw[i - n];
      V.Y2[2 * (i - n)] = yv;
      if (V.Yc) V.Yc[i - n] = yv;
      red[0] += r * r;
    }
  }
  if (grid_sum_last<1>(red, V.part, &c->counter) && threadIdx.x == 0) {
    if (defer) V.dred[0] = red[0];
    else prep_finish(c, red[0], variant, R);
  }
}
__global__ void k_prep_finish(Vec V, int variant, int R) {
  if (V.ctl->stop || threadIdx.x) return;
  prep_finish(V.ctl, V.dred[0], variant, R);
}

// Device-side loop control (build_loop_graph): the body of a WHILE graph
// node is [k_loop_pick -> SWITCH(non-refresh graph, refresh graph) ->
// k_loop_next].  k_loop_pick selects this iteration's variant from the
// refresh schedule (k_sched = 1, 1 + R, ...); k_loop_next counts the
// iteration and keeps looping while iterations are left and no kernel has
// stopped the solve (termination status, error).  One solve is one graph
// launch: no host synchronisation and no no-op iterations after the stop.
__global__ void k_loop_pick(Ctl* c, cudaGraphConditionalHandle sw, int R) {
  const bool refresh = R > 0 && c->k_sched % R == 0;  // before k_prep's increment
  if (refresh) c->loop_refresh += 1;
  cudaGraphSetConditional(sw, refresh ? 1u : 0u);
}
__global__ void k_loop_next(Ctl* c, cudaGraphConditionalHandle wh) {
  c->loop_done += 1;
  c->loop_left -= 1;
  cudaGraphSetConditional(wh, (c->loop_left > 0 && !c->stop) ? 1u : 0u);
}

// x += alpha p; r -= alpha Gp; r'r -> stop test / beta (sparse_linalg.py:279-288).
// Opt-in PCG: beta from r'M^-1 r.  Opt-in recurrence (recur): A x is carried
// as Axw += alpha q over the m rows (the final A pass is then skipped).
__global__ void __launch_bounds__(kBlock) k_cg_update(Vec V, long long cap, int recur) {
  Ctl* c = V.ctl;
  if (c->stop || c->cg_done) return;
  const double a = c->cg_alpha;
  double red[2] = {0.0, 0.0};
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  for (long long j = tid; j < V.n; j += nt) {
    if (V.T) V.T[j] += a * V.AtAp[j];  // A^T A x += alpha A^T A p
    V.x[j] += a * V.X2[2 * j];
    const double r = V.r[j] - a * V.Gp[j];
    V.r[j] = r;
    red[0] += r * r;
    if (V.Minv) red[1] += r * (V.Minv[j] * r);
  }
  if (recur)
    for (long long i = tid; i < V.m; i += nt) V.Axw[i] += a * V.q[i];
  if (grid_sum_last<2>(red, V.part, &c->counter) && threadIdx.x == 0) {
    c->cg_it += 1;
    const double rs_new = red[0];
    if (!isfinite(rs_new)) { c->err |= ERR_CG_NONFINITE; c->stop = 1; c->cg_done = 1; return; }
    if (sqrt(rs_new) <= c->tol || c->cg_it >= cap) { c->cg_done = 1; return; }
    const double rb = V.Minv ? red[1] : rs_new;
    c->cg_beta = rb / c->rs;
    c->rs = rb;
  }
}

// p = r + beta p (sparse_linalg.py:287); PCG: p = M^-1 r + beta p
__global__ void __launch_bounds__(kBlock) k_cg_p(Vec V) {
  Ctl* c = V.ctl;
  if (c->stop || c->cg_done) return;
  const double be = c->cg_beta;
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  if (V.Minv)
    for (long long j = tid; j < V.n; j += nt) {
      const double pj = V.Minv[j] * V.r[j] + be * V.X2[2 * j];
      V.X2[2 * j] = pj;
      V.P1[j] = pj;
    }
  else
    for (long long j = tid; j < V.n; j += nt) {
      const double pj = V.r[j] + be * V.X2[2 * j];
      V.X2[2 * j] = pj;
      V.P1[j] = pj;
    }
}

// relaxed point of element i of the (x, y) part:
//   u~ = p - corr g (embedding.py:193), u_bar = alpha u~ + (1-alpha) u
//   (solver.py:163), t = u_bar - v (cone input, solver.py:164)
struct Relax {
  double ut, ub, t;
};
__device__ __forceinline__ Relax relax_y(const Vec& V, long long i, double corr, double al) {
  Relax r;
  r.ut = V.zy[i] - corr * V.gy[i];
  r.ub = al * r.ut + (1.0 - al) * V.u[V.n + i];
  r.t = r.ub - V.v[V.n + i];
  return r;
}
__device__ __forceinline__ void store_y(const Vec& V, long long i, double ub, double up) {
  const double vi = V.v[V.n + i];
  V.u[V.n + i] = up;
  V.Y2[2 * i + 1] = up;           // gather copy for the next residual pass
  V.v[V.n + i] = (vi - ub) + up;  // solver.py:165
}

__device__ __forceinline__ void soc_factor(double nz, double t, double* mode, double* head,
                                           double* scale) {
  // cones.py:172-184
  if (nz <= -t) { *mode = 0.0; *head = 0.0; *scale = 0.0; }
  else if (nz <= t) { *mode = 1.0; *head = t; *scale = 1.0; }
  else {
    const double a = 0.5 * (nz + t);
    *mode = 2.0; *head = a; *scale = a / nz;
  }
}

// Affine tail + relaxation + cone projection of every block that one warp
// or thread can finish alone (x-part free, zero, nonneg, small SOC, exp),
// plus big-SOC chunk norms; the last block sets the tau entries, the big
// SOC factors and the iteration counter.
// tau entry (embedding.py:196, cones.py:248), iteration counter, and the
// big-SOC factors (cones.py:172-184) from the (all-reduced) cone_red totals.
// Runs in the last block of k_cone_tail, or as k_cone_finish after the
// all-reduce when rows are sharded.
__device__ void cone_finish(Vec V, Cones K) {
  Ctl* c = V.ctl;
  const double* cr = V.cone_red;
  const long long n = V.n, m = V.m;
  const double al = c->alpha;
  if (threadIdx.x == 0) {
    if (cr[2] != 0.0) { c->err |= ERR_CONE_NONFINITE; c->stop = 1; }
    const double ut_ = V.u[n + m], vt_ = V.v[n + m];
    const double wt = ut_ + vt_;
    const double utau = (wt + cr[0]) + cr[1];
    const double ub = al * utau + (1.0 - al) * ut_;
    const double t = ub - vt_;
    if (!isfinite(t)) { c->err |= ERR_CONE_NONFINITE; c->stop = 1; }
    const double up = fmax(t, 0.0);
    V.u[n + m] = up;
    V.v[n + m] = (vt_ - ub) + up;
    c->iter += 1;
    c->check_pending = (c->iter % c->check_interval == 0);  // solver.py:359
  }
  for (int q = threadIdx.x; q < K.n_bsoc; q += blockDim.x) {
    const int g = K.bsoc_gid[q];
    soc_factor(sqrt(cr[3 + 2 * g]), cr[4 + 2 * g], V.soc_fac + 3 * q, V.soc_fac + 3 * q + 1,
               V.soc_fac + 3 * q + 2);
  }
}

__global__ void k_cone_finish(Vec V, Cones K) {
  if (V.ctl->stop) return;
  cone_finish(V, K);
}

// (64-register cap: 4 CTAs per SM instead of 3 -- config 5's streaming
// loops 228 -> 197 us; a 40-register cap spills and is slower)
__global__ void __launch_bounds__(kBlock, 4) k_cone_tail(Vec V, Cones K, int defer) {
  Ctl* c = V.ctl;
  if (c->stop) return;
  const long long n = V.n, m = V.m;
  const double corr = c->corr, al = c->alpha;
  double red[2] = {0.0, 0.0};  // c'u~_x, b'u~_y
  int bad = 0;
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  // x-part: free cone (cones.py:246); v_x becomes exactly 0
  for (long long j = tid; j < n; j += nt) {
    const double ut = V.x[j] - corr * V.gx[j];
    red[0] += V.xw * (V.c[j] * ut);
    const double ub = al * ut + (1.0 - al) * V.u[j];
    const double t = ub - V.v[j];
    bad |= !isfinite(t);
    const double vj = V.v[j];
    V.u[j] = t;
    V.X2[2 * j + 1] = t;
    V.v[j] = (vj - ub) + t;
    if (V.T) {  // A^T (v+_y - u+_y) = A^T v_y - A^T u_bar_y, u~_y = z_y - corr g_y
      const double aut = (V.Sv[j] + V.T[j]) - corr * V.Atgy[j];
      const double uyj = V.Uy[j];
      V.Dd[j] = (V.Dd[j] + uyj) - (al * aut + (1.0 - al) * uyj);
    }
  }
  // residual recurrence: v_x == 0, so u+_x = al (x - corr g_x) + (1 - al) u_x
  // and A u+_x = al (A x - corr A g_x) + (1 - al) A u_x (all terms on hand:
  // A x from the final CG pass, A g_x from setup); refreshed directly every
  // R iterations by the merged first CG pass
  if (V.Agx)
    for (long long i = tid; i < m; i += nt)
      V.Aux[i] = al * (V.Axw[i] - corr * V.Agx[i]) + (1.0 - al) * V.Aux[i];
  // zero (free in K*) and nonnegative rows
  const long long zl = K.z + K.l;
  for (long long i = tid; i < zl; i += nt) {
    const Relax r = relax_y(V, i, corr, al);
    red[1] += V.b[i] * r.ut;
    bad |= !isfinite(r.t);
    store_y(V, i, r.ub, i < K.z ? r.t : fmax(r.t, 0.0));
  }
  // PSD and big-SOC rows only contribute b'u~ here (projected in k_cone_apply)
  for (long long i = K.psd_lo + tid; i < K.psd_hi; i += nt) {
    const Relax r = relax_y(V, i, corr, al);
    red[1] += V.b[i] * r.ut;
    bad |= !isfinite(r.t);
  }
  // small SOCs: one warp per cone
  {
    const int lane = threadIdx.x & 31;
    const long long warp = tid >> 5, nw = nt >> 5;
    for (long long q = warp; q < K.n_ssoc; q += nw) {
      const long long o = K.ssoc_off[q], d = K.ssoc_len[q];
      double zz = 0.0, t0 = 0.0, part = 0.0;
      for (long long e = lane; e < d; e += 32) {
        const Relax r = relax_y(V, o + e, corr, al);
        part += V.b[o + e] * r.ut;
        bad |= !isfinite(r.t);
        if (e == 0) t0 = r.t; else zz += r.t * r.t;
      }
      red[1] += part;
      zz = warp_sum(zz);
      t0 = __shfl_sync(0xffffffffu, t0, 0);
      double mode, head, scale;
      soc_factor(sqrt(zz), t0, &mode, &head, &scale);
      for (long long e = lane; e < d; e += 32) {
        const Relax r = relax_y(V, o + e, corr, al);
        double up;
        if (mode == 0.0) up = 0.0;
        else if (mode == 1.0) up = r.t;
        else up = (e == 0) ? head : scale * r.t;
        store_y(V, o + e, r.ub, up);
      }
    }
  }
  // exponential cones: one thread per cone, K_exp* (dual) projection
  for (long long q = tid; q < K.n_exp; q += nt) {
    const long long o = K.exp_lo + 3 * q;
    double tv[3], ub[3], pr[3];
    for (int e = 0; e < 3; ++e) {
      const Relax r = relax_y(V, o + e, corr, al);
      red[1] += V.b[o + e] * r.ut;
      bad |= !isfinite(r.t);
      tv[e] = r.t;
      ub[e] = r.ub;
    }
    exp_proj_dual(tv, pr);
    for (int e = 0; e < 3; ++e) store_y(V, o + e, ub[e], pr[e]);
  }
  // big SOC chunks: one block per chunk -> partial ||z||^2 (head excluded)
  for (long long ch = blockIdx.x; ch < K.n_chunk; ch += gridDim.x) {
    const long long o = K.chunk_off[ch];
    const int len = K.chunk_len[ch];
    const long long head = K.bsoc_off[K.chunk_cone[ch]];
    double zz[1] = {0.0};
    for (int e = threadIdx.x; e < len; e += kBlock) {
      const Relax r = relax_y(V, o + e, corr, al);
      red[1] += V.b[o + e] * r.ut;
      bad |= !isfinite(r.t);
      if (o + e != head) zz[0] += r.t * r.t;
    }
    block_sum<1>(zz);
    if (threadIdx.x == 0) V.chunk_part[ch] = zz[0];
  }
  // never flip `stop` outside a last block: blocks that had not started yet
  // would skip the reduction and strand its counter
  if (bad) atomicOr(&c->err, ERR_CONE_NONFINITE);
  if (!grid_sum_last<2>(red, V.part, &c->counter)) return;
  // ---- last block: local totals into cone_red ------------------------------
  double* cr = V.cone_red;
  if (threadIdx.x == 0) {
    cr[0] = red[0];
    cr[1] = red[1];
    cr[2] = (double)c->err;
  }
  for (int g = threadIdx.x; g < K.n_big_global; g += kBlock) {
    cr[3 + 2 * g] = 0.0;
    cr[4 + 2 * g] = 0.0;
  }
  __syncthreads();
  // big SOC partial norms: one warp per local cone over its chunk partials
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < K.n_bsoc; q += kWarps) {
    double zz = 0.0;
    for (int ch = K.bsoc_chunk_lo[q] + lane; ch < K.bsoc_chunk_lo[q + 1]; ch += 32)
      zz += __ldcg(V.chunk_part + ch);
    zz = warp_sum(zz);
    if (lane == 0) {
      const int g = K.bsoc_gid[q];
      cr[3 + 2 * g] = zz;
      if (K.bsoc_off[q] >= 0) cr[4 + 2 * g] = relax_y(V, K.bsoc_off[q], corr, al).t;  // head is local
    }
  }
  __syncthreads();
  if (!defer) cone_finish(V, K);
}

// Big SOC apply (block per chunk) and PSD blocks (block per PSD, Jacobi in
// shared memory, or in global scratch for sides beyond the smem budget).
// One PSD block (cones.py:147-191): unpack svec of the relaxed point (off-
// diagonals / sqrt 2), Jacobi, X = V diag(max(lambda, 0)) V^T repacked.
template <int KC, class G>
__device__ void psd_block(const G& g, const Vec& V, Ctl* c, long long o, int k_rt, double corr,
                          double al, double* M, double* Vv, double* cs, double* sn, int* pp,
                          int* qq, double* dpp, double* dqq) {
  const int k = KC > 0 ? KC : k_rt;
  const int len = k * (k + 1) / 2;
  for (int e = g.rank(); e < len; e += g.size()) {
    int i, j;
    svec_rc(e, k, i, j);
    const Relax r = relax_y(V, o + e, corr, al);
    const double val = (i == j) ? r.t : r.t / 1.4142135623730951;
    M[i * k + j] = val;
    M[j * k + i] = val;
  }
  g.sync();
  const bool ok = group_jacobi<KC>(g, M, Vv, k, cs, sn, pp, qq, dpp, dqq);
  if (!ok) {
    if (g.rank() == 0) {
      atomicOr(&c->err, ERR_JACOBI);
      if (V.dbg && atomicCAS(reinterpret_cast<unsigned long long*>(V.dbg), 0ull, 1ull) == 0ull) {
        V.dbg[1] = k;
        for (int e = 0; e < len; ++e) V.dbg[2 + e] = relax_y(V, o + e, corr, al).t;
      }
    }
    g.sync();
    return;
  }
  for (int e = g.rank(); e < len; e += g.size()) {
    int i, j;
    svec_rc(e, k, i, j);
    double x = 0.0;
    for (int t = 0; t < k; ++t) {
      const double lam = M[t * k + t];
      if (lam > 0.0) x += Vv[i * k + t] * lam * Vv[j * k + t];
    }
    const Relax r = relax_y(V, o + e, corr, al);
    store_y(V, o + e, r.ub, (i == j) ? x : x * 1.4142135623730951);
  }
  g.sync();
}

__global__ void __launch_bounds__(kBlock) k_cone_apply(Vec V, Cones K, double* psd_scratch,
                                                       int smem_side, const int* cta_list,
                                                       int n_cta) {
  Ctl* c = V.ctl;
  if (c->stop) return;
  const double corr = c->corr, al = c->alpha;
  for (long long ch = blockIdx.x; ch < K.n_chunk; ch += gridDim.x) {
    const long long o = K.chunk_off[ch];
    const int len = K.chunk_len[ch];
    const int q = K.chunk_cone[ch];
    const long long head = K.bsoc_off[q];
    const double mode = V.soc_fac[3 * q], hv = V.soc_fac[3 * q + 1], sc = V.soc_fac[3 * q + 2];
    for (int e = threadIdx.x; e < len; e += kBlock) {
      const Relax r = relax_y(V, o + e, corr, al);
      double up;
      if (mode == 0.0) up = 0.0;
      else if (mode == 1.0) up = r.t;
      else up = (o + e == head) ? hv : sc * r.t;
      store_y(V, o + e, r.ub, up);
    }
  }
  if (n_cta == 0) return;
  extern __shared__ double smem[];
  __shared__ double cs[128], sn[128], dpp[128], dqq[128];
  __shared__ int pp[128], qq[128];
  // blocks of side > kWarpPsd not on the cooperative grid: one CTA each (a
  // list -- r01 walked all blocks, and config 4's 11,111 warp-sized ones
  // cost each CTA ~75 dependent loads: 52 us for nothing)
  for (int t = blockIdx.x; t < n_cta; t += gridDim.x) {
    const int b = cta_list[t];
    const int k = K.psd_side[b];
    const long long o = K.psd_off[b];
    double* M;
    double* Vv;
    double *pcs = cs, *psn = sn, *pdp = dpp, *pdq = dqq;
    int *ppp = pp, *pqq = qq;
    if (k <= smem_side) { M = smem; Vv = smem + k * k; }
    else {  // matrices (and, beyond 128 rotation pairs, the pair arrays) in global scratch
      M = psd_scratch + K.psd_goff[b];
      Vv = M + (size_t)k * k;
      const int np = (k + 1) / 2;
      if (np > 128) {
        pcs = Vv + (size_t)k * k; psn = pcs + np; pdp = psn + np; pdq = pdp + np;
        ppp = reinterpret_cast<int*>(pdq + np); pqq = ppp + np;
      }
    }
    psd_block<0>(CtaGroup{}, V, c, o, k, corr, al, M, Vv, pcs, psn, ppp, pqq, pdp, pdq);
  }
}

// PSD blocks of side <= kWarpPsd: one warp each over a list of block
// indices (largest sides first), per-warp slices of the dynamic smem.
// (Measured on config 4's 11,111 blocks of side 3-8: a single launch with
// a warp per block beat 8- or 16-lane groups with one launch per side.
// r02 ncu: the kernel is issue-bound -- 72% of issue slots, FP64 12% of the
// instructions -- hence the per-side template bodies below.)
constexpr size_t kPsdSmallSmem = (size_t)(kBlock / 32) * 2 * kWarpPsd * kWarpPsd * sizeof(double);
__global__ void __launch_bounds__(kBlock, 4) k_psd_small(Vec V, Cones K, const int* list, int count) {
  Ctl* c = V.ctl;
  if (c->stop) return;
  const double corr = c->corr, al = c->alpha;
  extern __shared__ double smem[];
  constexpr int kW = kBlock / 32;
  __shared__ double wcs[kW][8], wsn[kW][8], wdp[kW][8], wdq[kW][8];
  __shared__ int wpp[kW][8], wqq[kW][8];
  const int wi = threadIdx.x >> 5;
  double* M = smem + (size_t)wi * 2 * kWarpPsd * kWarpPsd;
  for (long long t = (long long)blockIdx.x * kW + wi; t < count; t += (long long)gridDim.x * kW) {
    const int b = list[t];
    const int k = K.psd_side[b];
    // the side as a compile-time constant: the Jacobi's index arithmetic
    // (/ k, % k, the round-robin % (k - 1)) folds to multiplies -- with a
    // runtime side, integer division was most of the kernel's instructions
    // (config 4: IMAD/ISETP/I2F/F2I 40% of 129M, FP64 12%; issue slots 72%).
    // The unrolled bodies want 120 registers; capped at 64 (4 CTAs per SM,
    // as before) the kernel takes 127 us instead of 170 (uncapped: 158).
    switch (k) {
#define SCS_PSD_SIDE(KK)                                                                   \
  case KK:                                                                                 \
    psd_block<KK>(WarpGroup{}, V, c, K.psd_off[b], k, corr, al, M, M + k * k, wcs[wi], wsn[wi], \
                  wpp[wi], wqq[wi], wdp[wi], wdq[wi]);                                     \
    break;
      SCS_PSD_SIDE(2) SCS_PSD_SIDE(3) SCS_PSD_SIDE(4) SCS_PSD_SIDE(5) SCS_PSD_SIDE(6)
      SCS_PSD_SIDE(7) SCS_PSD_SIDE(8) SCS_PSD_SIDE(9) SCS_PSD_SIDE(10) SCS_PSD_SIDE(11)
      SCS_PSD_SIDE(12) SCS_PSD_SIDE(13) SCS_PSD_SIDE(14) SCS_PSD_SIDE(15) SCS_PSD_SIDE(16)
#undef SCS_PSD_SIDE
      default:
        psd_block<0>(WarpGroup{}, V, c, K.psd_off[b], k, corr, al, M, M + k * k, wcs[wi], wsn[wi],
                     wpp[wi], wqq[wi], wdp[wi], wdq[wi]);
    }
  }
}

// ---------------------------------------------------------------------------
// Large PSD blocks (side > the shared-memory side; RPCA's 2p x 2p block,
// generators.py:197-286): the whole cooperative grid works on one block at a
// time, M and V in global scratch (row-major, L2-resident up to side ~2500),
// two grid barriers per Jacobi round.  Same parallel (round-robin) order,
// tiny-entry rule and stopping test as group_jacobi (cones.cuh), which
// follows _kernels.py:137-191.  A round applies M <- J^T M J as independent
// 2x2-block updates: thread item (pi, pj) reads rows {p_i, q_i} x columns
// {p_j, q_j}, applies the column then the row rotation and writes them back
// in place (no other item touches those four entries), and item (i, pj)
// rotates columns p_j, q_j of row i of V.  Items whose two rotations are
// both the identity are skipped (most of them in the late sweeps).  Every
// CTA computes the round's rotation parameters for all pairs redundantly
// into shared memory from the diagonal blocks (a barrier then separates
// those reads from the diagonal-block writes).  Loads and stores go through L2 (__ldcg / __stcg): another SM
// wrote the data in the previous round.  The reconstruction
// X = V diag(max(lambda, 0)) V^T is a tiled fp64 product over the lower
// triangle of 64 x 64 tiles, written straight into svec order.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;
constexpr int kPsdTile = 64, kPsdTk = 32;
constexpr size_t kPsdTileSmem = (size_t)2 * kPsdTk * (kPsdTile + 1) * sizeof(double);
__host__ __device__ constexpr size_t psd_grid_pair_bytes(int k) {
  return (size_t)((k + 1) / 2) * (4 * sizeof(double) + 2 * sizeof(int));
}

// deterministic grid sum: per-CTA partials, barrier, every thread adds them
// in CTA order; a trailing barrier frees `part` for the next use
__device__ double psd_grid_sum(const cg::grid_group& grid, double v, double* part) {
  double a[1] = {v};
  block_sum<1>(a);
  if (threadIdx.x == 0) __stcg(part + blockIdx.x, a[0]);
  grid.sync();
  double t = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(part + b);
  grid.sync();
  return t;
}

__device__ __forceinline__ long long svec_index(int r, int col, int k) {
  // element (r, col), r >= col, of the column-major packed lower triangle
  return (long long)col * k - (long long)col * (col - 1) / 2 + (r - col);
}

__global__ void __launch_bounds__(kBlock, 2) k_psd_grid(Vec V, Cones K, double* psd_scratch,
                                                     const int* list, int count, double* part) {
  cg::grid_group grid = cg::this_grid();
  Ctl* c = V.ctl;
  if (c->stop) return;
  const double corr = c->corr, al = c->alpha;
  extern __shared__ double smem[];
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gsz = (long long)gridDim.x * blockDim.x;
  constexpr int kU = 4;
  for (int bi = 0; bi < count; ++bi) {
    const int b = list[bi];
    const int k = K.psd_side[b];
    const long long o = K.psd_off[b];
    double* M = psd_scratch + K.psd_goff[b];
    double* Vv = M + (size_t)k * k;
    double* lam = Vv + (size_t)k * k;
    // unpack the relaxed point (off-diagonals / sqrt 2) and V = I
    double fro = 0.0;
    for (long long w = gtid; w < (long long)k * k; w += gsz) {
      const int i = (int)(w / k), j = (int)(w % k);
      const long long e = i >= j ? svec_index(i, j, k) : svec_index(j, i, k);
      const double t = relax_y(V, o + e, corr, al).t;
      const double val = i == j ? t : t / 1.4142135623730951;
      __stcg(M + w, val);
      __stcg(Vv + w, i == j ? 1.0 : 0.0);
      fro += val * val;
    }
    fro = psd_grid_sum(grid, fro, part);
    if (!isfinite(fro)) {
      if (gtid == 0) atomicOr(&c->err, ERR_CONE_NONFINITE);
      continue;
    }
    const double thresh = 1e-12 * sqrt(fro);
    const double tiny = thresh / (2.0 * k);
    const int kk = k + (k & 1);
    const int np = kk / 2;
    double* cs = smem;
    double* sn = cs + np;
    double* dp = sn + np;
    double* dq = dp + np;
    int* pp = reinterpret_cast<int*>(dq + np);
    int* qq = pp + np;
    // item geometry: rpi row-items per thread pass when the pair count is
    // below the CTA size, else one row-item and a column loop
    const int rpi = np >= (int)blockDim.x ? 1 : (int)blockDim.x / np;
    const int rsub = rpi > 1 ? (int)threadIdx.x / np : 0;
    const int col0 = rpi > 1 ? (int)threadIdx.x - rsub * np : (int)threadIdx.x;
    const int cstep = rpi > 1 ? np : (int)blockDim.x;
    const int ngroup = (np + k + rpi - 1) / rpi;
    bool ok = k == 1;
    for (int sweep = 0; sweep <= 100 && !ok; ++sweep) {
      double off = 0.0;
      for (long long w = gtid; w < (long long)k * k; w += gsz) {
        const int i = (int)(w / k), j = (int)(w % k);
        if (j > i) { const double x = __ldcg(M + w); off += 2.0 * x * x; }
      }
      off = psd_grid_sum(grid, off, part);
      if (sqrt(off) <= thresh) { ok = true; break; }
      if (sweep == 100) break;
      for (int step = 0; step < kk - 1; ++step) {
        // rotation parameters of every pair (loads of kU pairs in flight)
        for (int p0 = threadIdx.x; p0 < np; p0 += kU * blockDim.x) {
          int pv[kU], qv[kU];
          double apq[kU], app[kU], aqq[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int pi = p0 + u * blockDim.x;
            pv[u] = 0; qv[u] = k;
            apq[u] = app[u] = aqq[u] = 0.0;
            if (pi < np) {
              const int a = rr_player(pi, step, kk), bb = rr_player(kk - 1 - pi, step, kk);
              pv[u] = a < bb ? a : bb; qv[u] = a < bb ? bb : a;
              if (qv[u] < k) {
                apq[u] = __ldcg(M + (size_t)pv[u] * k + qv[u]);
                app[u] = __ldcg(M + (size_t)pv[u] * k + pv[u]);
                aqq[u] = __ldcg(M + (size_t)qv[u] * k + qv[u]);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int pi = p0 + u * blockDim.x;
            if (pi >= np) continue;
            double cc = 1.0, ss = 0.0, vp = app[u], vq = aqq[u];
            if (qv[u] < k && fabs(apq[u]) > tiny) {
              const double tau = (aqq[u] - app[u]) / (2.0 * apq[u]);
              const double root = sqrt(1.0 + tau * tau);
              const double t = tau >= 0.0 ? 1.0 / (tau + root) : 1.0 / (tau - root);
              cc = 1.0 / sqrt(1.0 + t * t);
              ss = t * cc;
              vp = app[u] - t * apq[u];
              vq = aqq[u] + t * apq[u];
            }
            pp[pi] = pv[u]; qq[pi] = qv[u]; cs[pi] = cc; sn[pi] = ss; dp[pi] = vp; dq[pi] = vq;
          }
        }
        // the diagonal-block items below overwrite the entries the other
        // CTAs read for these parameters
        grid.sync();
        // items: row-items ri < np are M block-rows pi = ri, the rest V rows
        // i = ri - np; a thread keeps one pair column pj and takes kU
        // row-items of its CTA's interleaved row groups at a time, all loads
        // of the batch before any store (items are disjoint)
        for (int pj = col0; rsub < rpi && pj < np; pj += cstep) {
          const double sj = sn[pj], cj = cs[pj];
          const int r = pp[pj], sc = qq[pj];
          const bool sok = sc < k;
          for (int g0 = blockIdx.x; g0 < ngroup; g0 += kU * (int)gridDim.x) {
            int kind[kU], off[kU][4];
            double x[kU][4], ci[kU], si[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              const int g = g0 + u * (int)gridDim.x;
              const int ri = g * rpi + rsub;
              kind[u] = 0;
              if (g >= ngroup || ri >= np + k) continue;
              if (ri < np) {
                const int pi = ri;
                const int p = pp[pi], q = qq[pi];
                if (pi == pj) {  // diagonal block: eigenvalue estimates, zero coupling
                  if (q < k) {
                    if (sn[pi] != 0.0) {
                      __stcg(M + (size_t)p * k + p, dp[pi]);
                      __stcg(M + (size_t)q * k + q, dq[pi]);
                    }
                    __stcg(M + (size_t)p * k + q, 0.0);
                    __stcg(M + (size_t)q * k + p, 0.0);
                  }
                  continue;
                }
                si[u] = sn[pi];
                if (si[u] == 0.0 && sj == 0.0) continue;
                ci[u] = cs[pi];
                const bool qok = q < k;
                kind[u] = 1;
                off[u][0] = p * k + r;
                off[u][1] = sok ? p * k + sc : -1;
                off[u][2] = qok ? q * k + r : -1;
                off[u][3] = (qok && sok) ? q * k + sc : -1;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  x[u][e] = off[u][e] >= 0 ? __ldcg(M + off[u][e]) : 0.0;
              } else {
                if (sj == 0.0) continue;
                const int i = ri - np;
                si[u] = 0.0; ci[u] = 1.0;
                kind[u] = 2;
                off[u][0] = i * k + r;
                off[u][1] = i * k + sc;
                off[u][2] = off[u][3] = -1;
                x[u][0] = __ldcg(Vv + off[u][0]);
                x[u][1] = __ldcg(Vv + off[u][1]);
                x[u][2] = x[u][3] = 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
              if (kind[u] == 0) continue;
              double b00 = x[u][0], b01 = x[u][1], b10 = x[u][2], b11 = x[u][3];
              if (sj != 0.0) {  // columns r, s
                const double t00 = cj * b00 - sj * b01, t01 = sj * b00 + cj * b01;
                const double t10 = cj * b10 - sj * b11, t11 = sj * b10 + cj * b11;
                b00 = t00; b01 = t01; b10 = t10; b11 = t11;
              }
              if (si[u] != 0.0) {  // rows p, q
                const double t00 = ci[u] * b00 - si[u] * b10, t10 = si[u] * b00 + ci[u] * b10;
                const double t01 = ci[u] * b01 - si[u] * b11, t11 = si[u] * b01 + ci[u] * b11;
                b00 = t00; b01 = t01; b10 = t10; b11 = t11;
              }
              double* base = kind[u] == 1 ? M : Vv;
              __stcg(base + off[u][0], b00);
              if (off[u][1] >= 0) __stcg(base + off[u][1], b01);
              if (off[u][2] >= 0) __stcg(base + off[u][2], b10);
              if (off[u][3] >= 0) __stcg(base + off[u][3], b11);
            }
          }
        }
        grid.sync();
      }
    }
    if (!ok) {
      if (gtid == 0) atomicOr(&c->err, ERR_JACOBI);
      continue;
    }
    for (long long t = gtid; t < k; t += gsz) {
      const double x = __ldcg(M + (size_t)t * k + t);
      __stcg(lam + t, x > 0.0 ? x : 0.0);
    }
    grid.sync();
    // X = V diag(lam+) V^T over lower-triangle tiles: As = (V lam) rows of
    // tile ti, Bs = V rows of tile tj, k-chunks of kPsdTk
    const int nt = (k + kPsdTile - 1) / kPsdTile;
    const long long ntiles = (long long)nt * (nt + 1) / 2;
    double (*As)[kPsdTile + 1] = reinterpret_cast<double (*)[kPsdTile + 1]>(smem);
    double (*Bs)[kPsdTile + 1] = As + kPsdTk;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
    for (long long tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
      int ti = (int)((sqrt(8.0 * (double)tl + 1.0) - 1.0) / 2.0);
      while ((long long)(ti + 1) * (ti + 2) / 2 <= tl) ++ti;
      while ((long long)ti * (ti + 1) / 2 > tl) --ti;
      const int tj = (int)(tl - (long long)ti * (ti + 1) / 2);
      const int r0 = ti * kPsdTile, c0 = tj * kPsdTile;
      double acc[4][4] = {};
      for (int t0 = 0; t0 < k; t0 += kPsdTk) {
        __syncthreads();
        for (int e = threadIdx.x; e < kPsdTk * kPsdTile; e += blockDim.x) {
          const int rr = e / kPsdTk, tt = e % kPsdTk;
          const int t = t0 + tt;
          const bool tin = t < k;
          const int gi = r0 + rr, gj = c0 + rr;
          As[tt][rr] = (tin && gi < k) ? __ldcg(Vv + (size_t)gi * k + t) * __ldcg(lam + t) : 0.0;
          Bs[tt][rr] = (tin && gj < k) ? __ldcg(Vv + (size_t)gj * k + t) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int tt = 0; tt < kPsdTk; ++tt) {
          double a[4], bv[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) { a[x] = As[tt][ty + 16 * x]; bv[x] = Bs[tt][tx + 16 * x]; }
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], bv[y], acc[x][y]);
        }
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int i = r0 + ty + 16 * x, j = c0 + tx + 16 * y;
          if (i >= k || j >= k || i < j) continue;
          const long long e = o + svec_index(i, j, k);
          const Relax r = relax_y(V, e, corr, al);
          store_y(V, e, r.ub, i == j ? acc[x][y] : acc[x][y] * 1.4142135623730951);
        }
    }
    grid.sync();
  }
}

__device__ void finish_residuals(Ctl* c, double ut, double s_pri, double s_unb, double buy,
                                 double s_dual, double s_inf, double cux) {
  // scaling.py:171-206
  const double unbdd = cux < 0.0 ? sqrt(s_unb) * c->c_ref / (-cux) : INFINITY;
  const double infeas = buy < 0.0 ? sqrt(s_inf) * c->b_ref / (-buy) : INFINITY;
  double pri, dual, gap, gth;
  if (ut > 0.0) {
    pri = sqrt(s_pri) / c->sigma;
    dual = sqrt(s_dual) / c->rho;
    const double ctx = cux / ut / (c->rho * c->sigma);
    const double bty = buy / ut / (c->rho * c->sigma);
    gap = ctx + bty;
    gth = 1.0 + fabs(ctx) + fabs(bty);
  } else {
    pri = dual = gap = INFINITY;
    gth = 1.0;
  }
  double* r = c->res;
  r[0] = pri; r[1] = dual; r[2] = gap;
  r[3] = 1.0 + c->b_norm; r[4] = 1.0 + c->c_norm; r[5] = gth;
  r[6] = unbdd; r[7] = infeas;
  if (c->force_check) return;
  // check_termination (solver.py:219-234)
  int st = SCS_RUNNING;
  if (pri <= c->eps[0] * r[3] && dual <= c->eps[1] * r[4] && fabs(gap) <= c->eps[2] * gth) {
    st = SCS_SOLVED;
  } else {
    const bool inf = infeas <= c->eps[3], unb = unbdd <= c->eps[4];
    if (inf && unb) st = SCS_INFEASIBLE_AND_UNBOUNDED;
    else if (inf) st = SCS_INFEASIBLE;
    else if (unb) st = SCS_UNBOUNDED;
  }
  if (st != SCS_RUNNING) { c->status = st; c->stop = 1; }
}

// ===========================================================================
// setup kernels
// ===========================================================================
__global__ void k_i64_to_i32(const long long* in, int* out, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = (int)in[i];
}
__global__ void k_iota(int* out, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = (int)i;
}
// column index of every CSC entry: one warp per column
__global__ void k_expand_cols(const long long* colptr, long long ncols, int* out) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long j = w; j < ncols; j += nw)
    for (long long k = colptr[j] + lane; k < colptr[j + 1]; k += 32) out[k] = (int)j;
}
// row pointer from sorted row keys: rp[i] = lower_bound(keys, i)
__global__ void k_rowptr(const int* keys, long long nnz, long long rows, long long* rp) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i <= rows; i += nt) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (keys[mid] < i) lo = mid + 1; else hi = mid;
    }
    rp[i] = lo;
  }
}
__global__ void k_gather_csr(const int* perm, const int* colidx, const double* vals, long long nnz,
                             int* ci, double* av) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt) {
    const int s = perm[k];
    ci[k] = colidx[s];
    av[k] = vals[s];
  }
}
// per-row Euclidean norm (scaling.py:96-100), warp per row
__global__ void k_row_norms(Csr A, double* out) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = w; r < A.rows; r += nw) {
    double s = 0.0;
    for (long long k = A.rp[r] + lane; k < A.rp[r + 1]; k += 32) s += A.v[k] * A.v[k];
    s = warp_sum(s);
    if (lane == 0) out[r] = sqrt(s);
  }
}
// per-row sum of squares (column norms of A come from CSR(A^T) rows; when
// rows are sharded these partial sums are all-reduced before the sqrt)
__global__ void k_row_sumsq(Csr A, double* out) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = w; r < A.rows; r += nw) {
    double s = 0.0;
    for (long long k = A.rp[r] + lane; k < A.rp[r + 1]; k += 32) s += A.v[k] * A.v[k];
    s = warp_sum(s);
    if (lane == 0) out[r] = s;
  }
}
// nrm = sqrt(sumsq); scale = where(nrm > 0, 1/sqrt(nrm), 1); acc *= scale
// (scaling.py:97, 405-407)
__global__ void k_inv_sqrt_scale(double* sumsq, long long n, double* scale, double* acc) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) {
    const double v = sqrt(sumsq[i]);
    sumsq[i] = v;
    const double s = v > 0.0 ? 1.0 / sqrt(v) : 1.0;
    scale[i] = s;
    acc[i] *= s;
  }
}
// v[k] *= s[row(k)] over a CSR (warp per row)
__global__ void k_scale_rows(long long* rp, double* v, long long rows, const double* s) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = w; r < rows; r += nw) {
    const double f = s[r];
    for (long long k = rp[r] + lane; k < rp[r + 1]; k += 32) v[k] *= f;
  }
}
// v[k] *= s[ci[k]] (column scaling of a CSR)
__global__ void k_scale_cols(const int* ci, double* v, long long nnz, const double* s) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long k = tid; k < nnz; k += nt) v[k] *= s[ci[k]];
}
// Row-block means (scaling.py:74-76, 409-413).  Every non-singleton
// cone block is a segment with a global id; each shard sums the row norms
// of its part into seg_sum[gid] (all-reduced when sharded), the mean is
// seg_sum / global length.  Singleton (zero/nonneg) rows keep their norm.
__global__ void k_seg_partial(const double* rn, int nseg, const long long* seg_off,
                              const long long* seg_len, const int* seg_gid, double* seg_sum) {
  for (int q = blockIdx.x; q < nseg; q += gridDim.x) {
    const long long o = seg_off[q], d = seg_len[q];
    double s[1] = {0.0};
    for (long long e = threadIdx.x; e < d; e += blockDim.x) s[0] += rn[o + e];
    block_sum<1>(s);
    if (threadIdx.x == 0) seg_sum[seg_gid[q]] = s[0];
  }
}
__global__ void k_seg_means(const double* seg_sum, const long long* glen, int nseg_g,
                            double* mean) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int g = tid; g < nseg_g; g += gridDim.x * blockDim.x) mean[g] = seg_sum[g] / (double)glen[g];
}
__global__ void k_block_rows(const double* rn, long long zl, int nseg, const long long* seg_off,
                             const long long* seg_len, const int* seg_gid, const double* mean,
                             double* rscale, double* D) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < zl; i += nt) {
    const double t = rn[i];
    const double s = t > 0.0 ? 1.0 / sqrt(t) : 1.0;
    rscale[i] = s;
    D[i] *= s;
  }
  for (int q = blockIdx.x; q < nseg; q += gridDim.x) {
    const long long o = seg_off[q], d = seg_len[q];
    const double mm = mean[seg_gid[q]];
    const double f = mm > 0.0 ? 1.0 / sqrt(mm) : 1.0;
    for (long long e = threadIdx.x; e < d; e += blockDim.x) {
      rscale[o + e] = f;
      D[o + e] *= f;
    }
  }
}
// out[0] += sum of positive entries, out[1] += count of positive entries
__global__ void k_pos_mean(const double* x, long long n, double* part, unsigned* counter,
                           double* out) {
  double red[2] = {0.0, 0.0};
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  for (long long i = tid; i < n; i += nt)
    if (x[i] > 0.0) { red[0] += x[i]; red[1] += 1.0; }
  if (grid_sum_last<2>(red, part, counter) && threadIdx.x == 0) {
    out[0] = red[0];
    out[1] = red[1];
  }
}
// out = {||a*b||^2, ||c/d||^2 ...}: generic weighted square norm
//   mode 0: sum (a_i b_i)^2 ; mode 1: sum (a_i / b_i)^2 ; mode 2: sum a_i b_i
__global__ void k_norm2(const double* a, const double* b, long long n, int mode, double* part,
                        unsigned* counter, double* out) {
  double red[1] = {0.0};
  const long long tid = (long long)blockIdx.x * kBlock + threadIdx.x;
  const long long nt = (long long)gridDim.x * kBlock;
  for (long long i = tid; i < n; i += nt) {
    double t;
    if (mode == 0) { t = a[i] * b[i]; red[0] += t * t; }
    else if (mode == 1) { t = a[i] / b[i]; red[0] += t * t; }
    else red[0] += a[i] * b[i];
  }
  if (grid_sum_last<1>(red, part, counter) && threadIdx.x == 0) *out = red[0];
}
// out = (s * w) * x   (b_hat = sigma D b, c_hat = rho E c: scaling.py:128)
__global__ void k_scale_vec(const double* x, const double* w, double s, long long n, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = s * w[i] * x[i];
}
// Warm start (scaling.py:132-137, solver.py:128-150)
__global__ void k_init_state(Vec V, const double* wx, const double* wy, const double* ws,
                             double sigma, double rho) {
  const long long n = V.n, m = V.m;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n + m + 1; i += nt) {
    double u = 0.0, v = 0.0;
    if (wx) {
      if (i < n) u = sigma * wx[i] / V.E[i];
      else if (i < n + m) { u = rho * wy[i - n] / V.D[i - n]; v = sigma * V.D[i - n] * ws[i - n]; }
      else u = 1.0;
    } else if (i == n + m) {
      u = 1.0;
      v = 1.0;
    }
    V.u[i] = u;
    V.v[i] = v;
    if (i < n) { V.x[i] = 0.0; V.X2[2 * i] = 0.0; V.P1[i] = 0.0; V.X2[2 * i + 1] = u; }
    if (i >= n && i < n + m) {
      V.Y2[2 * (i - n)] = 0.0;
      V.Y2[2 * (i - n) + 1] = u;
      V.Axw[i - n] = 0.0;
    }
  }
}
// x / E  and y / D helpers for point residuals
__global__ void k_div(const double* a, const double* b, long long n, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = a[i] / b[i];
}
// residual vector pieces for _point_residuals: out_i = (a_i / w_i) + s_i - b_i
__global__ void k_point_pri(const double* ax, const double* D, const double* s, const double* b,
                            long long m, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < m; i += nt) out[i] = ax[i] / D[i] + s[i] - b[i];
}
// A x from the kept product of the final state: A_hat (x / E) = A_hat u_x / (tau sigma)
// (x = E (u_x / tau) / sigma, solver.py:262), likewise A_hat^T (y / D) = A_hat^T u_y / (tau rho)
__global__ void k_prod_scale(const double* prod, const double* utau, double scal, long long n,
                             double* out) {
  const double ut = *utau;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = prod[i] / ut / scal;
}
__global__ void k_point_dual(const double* aty, const double* E, const double* c, long long n,
                             double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = aty[i] / E[i] + c[i];
}
// Y2 for the setup solve: slot 0 = b_hat (rhs_y + A 0), slot 1 = 0
__global__ void k_fill_y2(double* Y2, const double* b, long long m) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < m; i += nt) { Y2[2 * i] = b[i]; Y2[2 * i + 1] = 0.0; }
}
__global__ void k_recip(const double* a, long long n, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) out[i] = 1.0 / a[i];
}
__global__ void k_sqrt(double* x, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) x[i] = sqrt(x[i]);
}
__global__ void k_add(double* a, const double* b, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) a[i] += b[i];
}
__global__ void k_zero(double* x, long long n) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) x[i] = 0.0;
}

}  // namespace scs

// ===========================================================================
// host side
// ===========================================================================
using namespace scs;

namespace {

std::mutex g_err_mu;
std::string g_err;

struct Timer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double s() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Fail {
  int code;
  std::string msg;
};

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw Fail{SCS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};        \
  } while (0)

// ---------------------------------------------------------------------------
// communicators for row sharding: NCCL (one process per GPU) or an
// in-process emulated group (several shards on one GPU, one host thread per
// shard) used to test the sharded kernels without a second GPU.  The
// emulated all-reduce synchronises on the host between kernels -- no kernel
// ever waits on another shard's kernel.
// ---------------------------------------------------------------------------
struct ScsComm {
  virtual ~ScsComm() {}
  virtual void allreduce(cudaStream_t st, double* d, size_t n) = 0;
  virtual bool capturable() const = 0;
};

}  // namespace

struct scs_emu_group {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool broken = false;
  std::vector<double*> ptr;
  std::vector<size_t> cnt;
};

namespace {

void emu_barrier(scs_emu_group* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->broken) throw Fail{SCS_ENCCL, "emulated group broken by another shard"};
  const long long my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    g->gen++;
    g->cv.notify_all();
    return;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->gen != my || g->broken; })) {
    g->broken = true;
    g->cv.notify_all();
    throw Fail{SCS_ENCCL, "emulated all-reduce timed out"};
  }
  if (g->broken) throw Fail{SCS_ENCCL, "emulated group broken by another shard"};
}

struct EmuComm : ScsComm {
  scs_emu_group* g;
  int rank;
  EmuComm(scs_emu_group* g_, int r) : g(g_), rank(r) {}
  void allreduce(cudaStream_t st, double* d, size_t n) override {
    CK(cudaStreamSynchronize(st));
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->ptr[rank] = d;
      g->cnt[rank] = n;
    }
    emu_barrier(g);
    if (rank == 0) {
      for (int r = 1; r < g->world; ++r)
        if (g->cnt[r] != n) throw Fail{SCS_ENCCL, "emulated all-reduce: count mismatch"};
      const int grid = (int)std::min<size_t>(1184, (n + 255) / 256 + 1);
      for (int r = 1; r < g->world; ++r) k_add<<<grid, 256, 0, st>>>(d, g->ptr[r], (long long)n);
      for (int r = 1; r < g->world; ++r)
        CK(cudaMemcpyAsync(g->ptr[r], d, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
    emu_barrier(g);
  }
  bool capturable() const override { return false; }
};

// One process per shard on one node, joined through a POSIX shared-memory
// segment (SCS_DIST_HOST): the all-reduce copies the buffer to this rank's
// slot, meets the others at a process-shared barrier, sums the slots in
// rank order (identical bits on every rank), and copies the sum back; big
// buffers go through in chunks.  Host-synchronised like EmuComm (not
// capturable): it exists to run the multi-process path -- bootstrap,
// per-rank generation, bounds -- where NCCL cannot (two ranks on one GPU).
struct ShmHeader {
  std::atomic<int> ready;
  std::atomic<int> broken;
  std::atomic<long long> arrived;
  std::atomic<long long> gen;
  int world;
  int pad;
  long long slot;  // doubles per rank slot
};
constexpr long long kShmSlot = 1 << 20;  // 8 MB per rank per chunk

struct ShmComm : ScsComm {
  ShmHeader* hd = nullptr;
  double* slots = nullptr;
  size_t bytes = 0;
  int rank = 0, world = 1;
  std::string name;
  std::vector<double> sum;
  ShmComm(const char* nm, int r, int w) : rank(r), world(w), name(nm) {
    bytes = sizeof(ShmHeader) + 64 + (size_t)w * kShmSlot * sizeof(double);
    int fd = -1;
    if (rank == 0) {
      shm_unlink(name.c_str());
      fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) throw Fail{SCS_ENCCL, "shm_open(create) " + name + ": " + strerror(errno)};
      if (ftruncate(fd, (off_t)bytes) != 0) {
        close(fd);
        throw Fail{SCS_ENCCL, std::string("ftruncate: ") + strerror(errno)};
      }
    } else {
      for (int t = 0; t < 12000 && fd < 0; ++t) {  // rank 0 creates it (<= 120 s)
        fd = shm_open(name.c_str(), O_RDWR, 0600);
        if (fd < 0) std::this_thread::sleep_for(std::chrono::milliseconds(10));
      }
      if (fd < 0) throw Fail{SCS_ENCCL, "shm_open " + name + ": " + strerror(errno)};
      struct stat stt;
      for (int t = 0; t < 12000; ++t) {
        if (fstat(fd, &stt) == 0 && (size_t)stt.st_size >= bytes) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
      }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Fail{SCS_ENCCL, std::string("mmap: ") + strerror(errno)};
    hd = reinterpret_cast<ShmHeader*>(p);
    slots = reinterpret_cast<double*>(reinterpret_cast<char*>(p) + sizeof(ShmHeader) + 64);
    if (rank == 0) {
      hd->world = w;
      hd->slot = kShmSlot;
      hd->arrived.store(0);
      hd->gen.store(0);
      hd->broken.store(0);
      hd->ready.store(1, std::memory_order_release);
    } else {
      for (int t = 0; t < 12000 && hd->ready.load(std::memory_order_acquire) != 1; ++t)
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
      if (hd->ready.load() != 1 || hd->world != w)
        throw Fail{SCS_ENCCL, "shared-memory group " + name + " not initialised for this world"};
    }
    cudaHostRegister(slots, (size_t)w * kShmSlot * sizeof(double), cudaHostRegisterDefault);
    cudaGetLastError();  // registration is an optimisation only
    barrier();           // every rank mapped before the first exchange
    if (rank == 0) shm_unlink(name.c_str());
  }
  ~ShmComm() override {
    if (hd) {
      cudaHostUnregister(slots);
      cudaGetLastError();
      munmap(hd, bytes);
    }
  }
  void barrier() {
    const long long my = hd->gen.load(std::memory_order_acquire);
    if (hd->arrived.fetch_add(1) + 1 == world) {
      hd->arrived.store(0);
      hd->gen.fetch_add(1, std::memory_order_release);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (long long spin = 0; hd->gen.load(std::memory_order_acquire) == my; ++spin) {
      if (hd->broken.load()) throw Fail{SCS_ENCCL, "shared-memory group broken by another rank"};
      if (spin > 1000) std::this_thread::sleep_for(std::chrono::microseconds(20));
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        hd->broken.store(1);
        throw Fail{SCS_ENCCL, "shared-memory all-reduce timed out"};
      }
    }
  }
  void allreduce(cudaStream_t st, double* d, size_t n) override {
    for (size_t off = 0; off < n || (n == 0 && off == 0); off += kShmSlot) {
      const size_t k = std::min<size_t>(kShmSlot, n - off);
      double* mine = slots + (size_t)rank * kShmSlot;
      if (k) CK(cudaMemcpyAsync(mine, d + off, k * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      barrier();
      sum.assign(k, 0.0);
      for (int r = 0; r < world; ++r) {
        const double* o = slots + (size_t)r * kShmSlot;
        if (r == 0) std::copy(o, o + k, sum.begin());
        else for (size_t i = 0; i < k; ++i) sum[i] += o[i];
      }
      barrier();  // slots free for the next chunk
      if (k) CK(cudaMemcpyAsync(d + off, sum.data(), k * sizeof(double), cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
      if (n == 0) break;
    }
  }
  bool capturable() const override { return false; }
};

#ifdef SCS_WITH_NCCL
struct NcclComm : ScsComm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  void allreduce(cudaStream_t st, double* d, size_t n) override {
    ncclResult_t r = ncclAllReduce(d, d, n, ncclDouble, ncclSum, c, st);
    if (r != ncclSuccess) throw Fail{SCS_ENCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r)};
  }
  bool capturable() const override { return true; }
};
#endif

}  // namespace

struct scs_handle {
  int dev = 0;
  int sms = 148;
  cudaStream_t st = nullptr;
  std::string err;
  // sizes
  long long m = 0, n = 0, nnz = 0, m_glob = 0, row_lo = 0;
  int rank = 0, world = 1;
  bool sharded = false;   // reductions over rows are all-reduced
  bool use_graph = true;  // iteration captured as a CUDA graph
  ScsComm* comm = nullptr;
  std::vector<long long> bounds;
  scs_settings set{};
  // matrices
  Csr A{}, At{};
  int LA = 32, LAt = 32;
  // TMA-streamed tiles (stream.cuh): format per matrix, schedules [matrix][pair]
  bool stm_m[2] = {false, false};
  Stm sF[2] = {};
  struct Sched {
    StmCmd* cmds = nullptr;
    long long* coff = nullptr;
    int G = 0, splits = 1;
    long long ncmd = 0;
  } ssch[2][2];
  double* Pstm = nullptr;
  unsigned long long stm_bytes[2] = {0, 0};
  // row-sharded: the A^T pass in row chunks, each chunk's all-reduce on a
  // second stream overlapping the next chunk's SpMV (SCS_AT_CHUNKS)
  static constexpr int kMaxChunks = 8;
  int at_chunks = 1;
  Sched at_sch[kMaxChunks][2];
  long long at_row[kMaxChunks + 1] = {};
  cudaStream_t st_comm = nullptr;
  cudaEvent_t ev_chunk[kMaxChunks] = {}, ev_comm = nullptr;
  bool stm_pair = false;  // NV = 1 passes on pair units sharing slab loads (SCS_STREAM_PAIR=1)
  int recur_refresh = 20;  // opt-in recurrence: direct A x every k iterations
  int res_rec = 32;        // A u_x of the residual check by recurrence, direct every k (0: always direct)
  bool res_rec_at = true;  // ... and A^T u_y (SCS_RES_RECUR_AT=0: only A u_x)
  // long rows split into pieces (setup_split): [A, A^T]
  bool split_m[2] = {false, false};
  Csr Asp[2] = {};
  int Lsp[2] = {2, 2};
  long long* seg[2] = {nullptr, nullptr};  // real row -> first piece (rows + 1)
  long long* long_rows[2] = {nullptr, nullptr};  // rows with > kLongSeg pieces
  long long n_long[2] = {0, 0};
  double* Psplit = nullptr;                // raw piece products (2 per piece)
  double* Minv = nullptr;  // opt-in PCG diagonal
  size_t l2_persist = 0, l2_window_max = 0;  // L2 set-aside for gather vectors
  // cones
  Cones K{};
  int nseg = 0, nseg_g = 0;
  long long* seg_off = nullptr;
  long long* seg_len = nullptr;
  int* seg_gid = nullptr;
  long long* seg_glen = nullptr;
  double* seg_sum = nullptr;
  double* seg_mean = nullptr;
  double* psd_scratch = nullptr;
  int smem_side = 0;
  int warp_side = kWarpPsd;  // PSD blocks up to this side: warp per block (SCS_PSD_WARP=0: off)
  int n_psd_small = 0;
  const int* psd_small_list = nullptr;  // their block indices, largest side first
  int n_psd_grid = 0;                   // blocks beyond smem_side: cooperative grid each
  const int* psd_grid_list = nullptr;
  int n_psd_cta = 0;                    // the others: one CTA each in k_cone_apply
  const int* psd_cta_list = nullptr;
  int psd_grid_ctas = 0;
  int psd_grid_max = 0;                 // largest side k_psd_grid takes (0: off)
  size_t psd_grid_smem = 0;
  double* psd_grid_part = nullptr;
  size_t cone_smem = 0;
  int cone_red_len = 3;
  // vectors
  Vec V{};
  double *b0 = nullptr, *c0 = nullptr;  // original b, c (device)
  double *bh = nullptr, *ch = nullptr, *D = nullptr, *E = nullptr;
  double *tmp_n = nullptr, *tmp_m = nullptr, *tmp_m2 = nullptr, *zero_m = nullptr;
  double* Traw = nullptr;   // raw A^T partial products (sharded)
  double* dscal = nullptr;  // device scratch scalars
  double* ext_y = nullptr;  // y of extract_point / point_residuals (m)
  Ctl* ctl = nullptr;
  Ctl* ctl_h = nullptr;     // pinned mirror
  double sigma = 1.0, rho = 1.0, mean_col = 1.0, mean_row = 1.0;
  double setup_seconds = 0.0;
  long long launches = 0, launches_per_iter = 0;
  long long launched_iters = 0;
  // iteration graph variants (build_graph): with the residual recurrences
  // on, a non-refresh (gvar[0]) and a refresh (gvar[1]) iteration, each
  // without the passes gated to the other kind; `variant` is the one being
  // enqueued (0: every pass, gated on the device)
  int variant = 0;
  int R = 0;                            // refresh period (0: one variant)
  cudaGraphExec_t gvar[2] = {nullptr, nullptr};
  long long lpi_var[2] = {0, 0};
  cudaGraphExec_t gloop = nullptr;      // device-side loop over the variants (one GPU)
  long long* loop_arg = nullptr;        // pinned: the iteration budget of a loop launch
  // V.Aux = A_hat u_x and V.Uy = A_hat^T u_y hold the products of the final
  // state (set by do_finish; the extraction then needs no matrix pass)
  bool prod_current = false;
  cudaStream_t st_copy = nullptr;       // extraction D2H overlapped with the point residuals
  void* stage_buf[2] = {nullptr, nullptr};  // pinned H2D staging during setup
  std::vector<DevBuf> bufs;
  int grid_full = 148 * 4;
};

namespace {

bool dbg_on() {
  static int on = -1;
  if (on < 0) on = getenv("SCS_DEBUG") ? 1 : 0;
  return on == 1;
}
void dbg(const char* fmt, ...) {
  if (!dbg_on()) return;
  static const auto t0 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  va_list ap;
  va_start(ap, fmt);
  fprintf(stderr, "[scs %9.1f ms] ", ms);
  vfprintf(stderr, fmt, ap);
  fprintf(stderr, "\n");
  fflush(stderr);
  va_end(ap);
}

void set_global_err(const std::string& s) {
  std::lock_guard<std::mutex> g(g_err_mu);
  g_err = s;
}

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// on the solver stream), which keeps freed blocks for reuse: the setup's
// multi-GB transients (radix-sort keys, permutations, format staging) are
// allocated and freed several times, and a plain cudaFree of such a block
// synchronises and unmaps (~1 s per setup at config 5).
template <class T>
T* dalloc(scs_handle* h, size_t count) {
  void* p = nullptr;
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T) + 16;  // +16: bulk-copy tails
  cudaError_t e = cudaMallocAsync(&p, bytes, h->st);
  if (e != cudaSuccess)
    throw Fail{SCS_ENOMEM, "cudaMallocAsync(" + std::to_string(bytes) + " bytes): " +
                               cudaGetErrorString(e)};
  h->bufs.push_back({p, bytes});
  return (T*)p;
}
void dfree(scs_handle* h, void* p) {
  if (!p) return;
  for (auto& b : h->bufs)
    if (b.p == p) { cudaFreeAsync(p, h->st); b.p = nullptr; }
}
// Large copies from pageable host memory (the caller's numpy arrays at
// setup: 16 GB at config 5): staged through two pinned 64-MB buffers that
// several host threads fill while the previous buffer's copy is in flight
// (pageable cudaMemcpy runs at a single staging thread's memcpy rate).
long long env_ll(const char* name, long long dflt);

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

void h2d_staged(scs_handle* h, void* dst, const void* src, size_t bytes) {
  constexpr size_t kChunk = 64ull << 20;
  static const int nthr = std::max(1, std::min(8, (int)std::thread::hardware_concurrency()));
  void** buf = h->stage_buf;  // allocated once per handle, freed at the end of setup
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (int i = 0; i < 2; ++i)
    if (!buf[i]) CK(cudaMallocHost(&buf[i], kChunk));
  CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  int k = 0;
  for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
    const size_t n = std::min(kChunk, bytes - off);
    CK(cudaEventSynchronize(ev[k]));  // the copy out of this buffer (two chunks ago) is done
    char* b = static_cast<char*>(buf[k]);
    const size_t per = (n + nthr - 1) / nthr;
    std::vector<std::thread> th;
    for (int t = 0; t < nthr; ++t) {
      const size_t a = std::min(n, t * per), e = std::min(n, a + per);
      if (e > a) th.emplace_back([=] { std::memcpy(b + a, s + off + a, e - a); });
    }
    for (auto& x : th) x.join();
    CK(cudaMemcpyAsync(d + off, b, n, cudaMemcpyHostToDevice, h->st));
    CK(cudaEventRecord(ev[k], h->st));
  }
  CK(cudaStreamSynchronize(h->st));
  for (int i = 0; i < 2; ++i) cudaEventDestroy(ev[i]);
}

void free_stage(scs_handle* h) {
  for (auto& b : h->stage_buf)
    if (b) { cudaFreeHost(b); b = nullptr; }
}

template <class T>
void h2d(scs_handle* h, T* dst, const T* src, size_t count) {
  static const bool staged = env_ll("SCS_H2D_STAGED", 1) != 0;
  if (staged && count * sizeof(T) >= (256ull << 20) && !host_pinned(src)) {
    h2d_staged(h, dst, src, count * sizeof(T));
    return;
  }
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, h->st));
}
template <class T>
void d2h(scs_handle* h, T* dst, const T* src, size_t count) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, h->st));
}

int elem_grid(scs_handle* h, long long work) {
  long long g = (work + kBlock - 1) / kBlock;
  return (int)std::max<long long>(1, std::min<long long>(g, h->grid_full));
}

// a pass gated to the other kind of iteration than the variant being enqueued
bool gated_off(const scs_handle* h, int rgate) {
  return (h->variant == 1 && rgate > 0) || (h->variant == 2 && rgate < 0);
}

// lanes per row: about 8 nonzeros per lane (two predicated 4-load steps)
int pick_lanes(long long nnz, long long rows) {
  const double avg = rows ? (double)nnz / (double)rows : 0.0;
  int L = 2;
  while (L < 32 && L * 8 < avg) L *= 2;
  return L;
}

void allreduce(scs_handle* h, double* d, size_t n) {
  if (h->sharded && n) h->comm->allreduce(h->st, d, n);
}

// A kernel's dynamic shared-memory ceiling is one attribute per device,
// shared by every handle in the process: it is raised once per (kernel,
// device) to the device's opt-in maximum and never lowered -- a handle
// setting its own, smaller need would break another handle's larger
// launches (two workspaces with different PSD sides on one GPU).  Returns
// the dynamic bytes available to the kernel.
int smem_optin(scs_handle* h, const void* fn) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(fn, h->dev);
  const auto it = done.find(key);
  if (it != done.end()) return it->second;
  int dev_optin = 0;
  CK(cudaDeviceGetAttribute(&dev_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  cudaFuncAttributes fa{};
  CK(cudaFuncGetAttributes(&fa, fn));
  const int avail = dev_optin - (int)fa.sharedSizeBytes;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, avail));
  done[key] = avail;
  return avail;
}

// CSR SpMV launch.  When the gathered vector is large (A^T passes of the
// 1e9-nonzero problem gather 80-160 MB, comparable to the 126 MB L2), the
// launch carries an L2 access-policy window marking it persisting, so the
// evict-first matrix stream cannot push it out (h->l2_persist bytes set
// aside at create; 0 = off).
template <int L, class Epi>
void launch_spmv_l(scs_handle* h, const Csr& M, const Epi& epi, int grid, size_t gbytes) {
  if (h->l2_persist == 0 || gbytes < ((size_t)16 << 20)) {
    k_spmv<L, Epi><<<grid, kBlock, 0, h->st>>>(M, epi);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = h->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow.base_ptr = (void*)epi.xb;
  at[0].val.accessPolicyWindow.num_bytes = std::min(gbytes, h->l2_window_max);
  at[0].val.accessPolicyWindow.hitRatio =
      (float)std::min(1.0, (double)h->l2_persist / (double)at[0].val.accessPolicyWindow.num_bytes);
  at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_spmv<L, Epi>, M, epi));
}

template <class Epi>
void launch_spmv(scs_handle* h, const Csr& M, int L, const Epi& epi) {
  const long long work = M.rows * (long long)L;
  const int grid = elem_grid(h, work);
  const long long gcols = (&M == &h->A) ? h->n : h->m;  // gathered vector length
  const size_t gbytes = (size_t)gcols * Epi::STRIDE * sizeof(double);
  switch (L) {
    case 2: launch_spmv_l<2, Epi>(h, M, epi, grid, gbytes); break;
    case 4: launch_spmv_l<4, Epi>(h, M, epi, grid, gbytes); break;
    case 8: launch_spmv_l<8, Epi>(h, M, epi, grid, gbytes); break;
    case 16: launch_spmv_l<16, Epi>(h, M, epi, grid, gbytes); break;
    default: launch_spmv_l<32, Epi>(h, M, epi, grid, gbytes); break;
  }
  h->launches++;
}

// Streamed-tile SpMV (stream.cuh).  NV = 1 passes run pair units (two
// sub-blocks share every slab load), NV = 2 passes single sub-blocks; the
// shared-memory ring gets as many 'cap'-byte stages (<= 4) as fit beside
// the accumulators and the two slab buffers.
// Returns the schedule's split count; with combine = false and splits > 1
// the split partials are left in Pstm for the caller's own epilogue kernel.
template <int NV, int STRIDE, class Epi>
int launch_stream(scs_handle* h, int mat, const Epi& epi, int chunk = -1, bool combine = true) {
  const Stm& F = h->sF[mat];
  const int pair = (NV == 1 && h->stm_pair) ? 1 : 0;  // NV = 1: pairs of sub-blocks share slab loads
  const auto& S = chunk < 0 ? h->ssch[mat][pair] : h->at_sch[chunk][pair];
  const long long r0 = chunk < 0 ? 0 : h->at_row[chunk], r1 = chunk < 0 ? F.rows : h->at_row[chunk + 1];
  const int accb = (pair ? 2 : 1) * kStmRS * NV * 8;
  const int optin = smem_optin(h, (const void*)k_stream<NV, STRIDE, Epi>);
  // two slab buffers (the next slab loads while the current one is read)
  // when at least 3 stages fit beside them, else one buffer (NV = 2 with
  // 4096-column slabs: 64 KB per slab)
  int NB = 2, NS = 0;
  size_t fixed = 0;
  for (; NB >= 1; --NB) {
    fixed = accb + (size_t)NB * F.W * STRIDE * 8 + kStmMaxStages * (2 * 8 + 16);
    NS = (int)std::min<long long>(kStmMaxStages, ((long long)optin - (long long)fixed) / F.cap);
    if (NS >= 3 || (NB == 1 && NS >= 2)) break;
  }
  if (NB < 1 || NS < 2) throw Fail{SCS_EINVAL, "streamed SpMV: shared memory budget exceeded"};
  const size_t smem = fixed + (size_t)NS * F.cap;
  const Csr& M = mat == 0 ? h->A : h->At;
  k_stream<NV, STRIDE, Epi><<<S.G, kStmThreads, smem, h->st>>>(F, S.cmds, S.coff, M, epi, S.splits,
                                                              h->Pstm, NS, NB, accb);
  CK(cudaGetLastError());
  h->launches++;
  // SCS_COMBINE_REPEAT=k (measurement only, tools/r02_combrep.sh): each
  // combine launched k times -- its in-graph cost is the slope of the
  // iteration time in k (the combines are idempotent but for statistics)
  static const int rep = (int)std::max<long long>(1, env_ll("SCS_COMBINE_REPEAT", 1));
  for (int r = 0; r < rep; ++r)
  if (S.splits > 1 && combine) {
    k_split_combine<Epi><<<elem_grid(h, r1 - r0), kBlock, 0, h->st>>>(h->Pstm, S.splits, F.rows, r0,
                                                                     r1, epi);
    h->launches++;
  }
  return S.splits;
}

// SpMV with the matrix A (mat = 0) or A^T (mat = 1): streamed tiles or the
// CSR kernel, as chosen at setup.
template <class Epi>
void launch_mat(scs_handle* h, int mat, const Epi& epi) {
  if (gated_off(h, epi.rgate)) return;
  if (h->stm_m[mat] && ((uintptr_t)epi.xb & 15) == 0) {
    launch_stream<Epi::NV, Epi::STRIDE, Epi>(h, mat, epi);
    return;
  }
  if (h->split_m[mat]) {  // long rows in pieces: raw piece products, then per-row sums
    EpiRaw<Epi> raw{};
    static_cast<Epi&>(raw) = epi;
    raw.T = h->Psplit;
    launch_spmv(h, h->Asp[mat], h->Lsp[mat], raw);
    const long long rows = mat == 0 ? h->m : h->n;
    k_rows<Epi><<<elem_grid(h, rows), kBlock, 0, h->st>>>(h->Psplit, rows, 1, epi, h->seg[mat],
                                                          h->long_rows[mat], h->n_long[mat]);
    h->launches++;
    return;
  }
  if (mat == 0) launch_spmv(h, h->A, h->LA, epi);
  else launch_spmv(h, h->At, h->LAt, epi);
}

template <class T>
void exclusive_scan(scs_handle* h, const T* in, T* out, long long n) {
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, h->st));
  void* tmp = dalloc<char>(h, bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, h->st));
  CK(cudaStreamSynchronize(h->st));
  dfree(h, tmp);
}

template <class T>
T read_dev(scs_handle* h, const T* p) {
  T v{};
  CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return v;
}

// ---------------------------------------------------------------------------
// TMA-streamed tiles (stream.cuh): format build and per-CTA schedules.
// ---------------------------------------------------------------------------
long long env_ll(const char* name, long long dflt) {
  const char* e = getenv(name);
  return e ? atoll(e) : dflt;
}

// Host-side tile table of one streamed matrix, kept only during setup.
struct StmTiles {
  int NB = 0, S = 0;
  std::vector<char> tiled;            // per sub-block: 1 tiled, 0 CSR
  std::vector<long long> pf;          // per tile: first piece (-1: none)
  std::vector<int> np;                // per tile: pieces
  std::vector<long long> slots;       // per tile
  std::vector<unsigned long long> poff;
  std::vector<unsigned> pslots;
  std::vector<long long> nnz_sb;      // per sub-block (CSR units' cost)
};

// Units -> LPT over persistent CTAs -> flat command lists (stream.cuh).
void build_stm_sched(scs_handle* h, int mat, int pair, const StmTiles& T, long long sb_lo,
                     long long sb_hi, scs_handle::Sched& S, int G0) {
  const Stm& F = h->sF[mat];
  struct Unit { long long sb0; int nsb; bool csr; int s_lo, s_hi, sp; double cost; };
  std::vector<Unit> units;
  long long ntiled = 0;
  for (long long sb = sb_lo; sb < sb_hi;) {
    if (!T.tiled[sb]) {
      units.push_back({sb, 1, true, 0, 0, 0, 0.0});
      ++sb;
      continue;
    }
    const int nsb = (pair && sb + 1 < sb_hi && T.tiled[sb + 1]) ? 2 : 1;
    units.push_back({sb, nsb, false, 0, T.S, 0, 0.0});
    ++ntiled;
    sb += nsb;
  }
  int splits = 1;
  // splits: the split count minimising (LPT makespan bound) + (split
  // partial rows written and read back by k_split_combine, + a launch)
  if (ntiled > 0) {
    double bytes = 0.0;
    for (long long t = sb_lo * T.S; t < sb_hi * T.S; ++t) bytes += 10.0 * (double)T.slots[t];
    const double part = 16.0 * (pair ? 1 : 2) * (double)F.rows;
    double best = 1e300;
    for (int sp = 1; sp <= std::min(32, std::max(1, T.S)); ++sp) {
      // longest-processing-time makespan <= average + largest unit
      const double U = (double)ntiled * sp;
      const double t = (bytes / G0 + bytes / U) / (6.0e12 / G0) +
                       (sp > 1 ? part * sp / 5.0e12 + 5e-6 : 0.0);
      if (t < best * 0.99) { best = t; splits = sp; }
    }
  }
  splits = (int)env_ll("SCS_STREAM_SPLITS", splits);
  splits = (int)env_ll(mat == 0 ? "SCS_STREAM_SPLITS_A" : "SCS_STREAM_SPLITS_AT", splits);
  splits = std::max(1, std::min(splits, std::max(1, T.S)));
  if (splits > 255) splits = 255;
  const double slab_cost = (double)F.W * 8.0 * (pair ? 1.5 : 2.0);
  std::vector<Unit> all;
  for (const Unit& u : units) {
    if (u.csr) {
      Unit v = u;
      v.cost = 44.0 * (double)T.nnz_sb[u.sb0] + 16.0 * kStmRS + 2e4;
      all.push_back(v);
      continue;
    }
    // per-slab slots of this unit, split into `splits` equal-slot slab ranges
    std::vector<double> cum(T.S + 1, 0.0);
    std::vector<int> nslab(T.S + 1, 0);
    for (int s = 0; s < T.S; ++s) {
      double a = 0.0;
      bool any = false;
      for (int q = 0; q < u.nsb; ++q) {
        const long long t = (u.sb0 + q) * T.S + s;
        a += 10.0 * (double)T.slots[t] + 2048.0 * T.np[t];  // + per-stage overhead
        any = any || T.np[t] > 0;
      }
      cum[s + 1] = cum[s] + a + (any ? slab_cost : 0.0);
    }
    int lo = 0;
    for (int sp = 0; sp < splits; ++sp) {
      int hi = T.S;
      if (sp + 1 < splits) {
        const double target = cum[T.S] * (sp + 1) / splits;
        hi = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        hi = std::max(lo, std::min(hi, T.S));
      }
      Unit v = u;
      v.s_lo = lo;
      v.s_hi = hi;
      v.sp = sp;
      v.cost = cum[hi] - cum[lo] + 2e4 * u.nsb;
      all.push_back(v);
      lo = hi;
    }
  }
  const int G = (int)std::max<long long>(1, std::min<long long>(G0, (long long)all.size()));
  std::vector<int> ord(all.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return all[a].cost > all[b].cost; });
  std::vector<std::vector<int>> cta(G);
  std::priority_queue<std::pair<double, int>, std::vector<std::pair<double, int>>,
                      std::greater<std::pair<double, int>>> pq;
  for (int g = 0; g < G; ++g) pq.push({0.0, g});
  for (int i : ord) {
    auto top = pq.top();
    pq.pop();
    cta[top.second].push_back(i);
    pq.push({top.first + all[i].cost, top.second});
  }
  // each CTA's parts in slab-range order (SCS_STREAM_ORDER=1), so that the
  // CTAs sweep the gathered vector's slab ranges roughly together
  if (splits > 1 && env_ll("SCS_STREAM_ORDER", 1))
    for (auto& l : cta)
      std::stable_sort(l.begin(), l.end(), [&](int a, int b) { return all[a].s_lo < all[b].s_lo; });
  std::vector<StmCmd> cmds;
  std::vector<long long> coff(G + 1, 0);
  for (int g = 0; g < G; ++g) {
    coff[g] = (long long)cmds.size();
    for (int ui : cta[g]) {
      const Unit& u = all[ui];
      const size_t first = cmds.size();
      const unsigned short pf = (unsigned short)(u.nsb == 2 ? STM_PAIR : 0);
      if (u.csr) {
        StmCmd c{};
        c.row0 = u.sb0 * kStmRS;
        c.flags = STM_CSR | STM_END;
        if (T.nnz_sb[u.sb0] > 16LL * kStmRS) c.flags |= STM_CSR32;  // long rows: warp per row
        cmds.push_back(c);
        continue;
      }
      for (int s = u.s_lo; s < u.s_hi; ++s)
        for (int q = 0; q < u.nsb; ++q) {
          const long long t = (u.sb0 + q) * T.S + s;
          for (int j = 0; j < T.np[t]; ++j) {
            const long long p = T.pf[t] + j;
            StmCmd c{};
            c.off = T.poff[p];
            c.bytes = (unsigned)stm_piece_bytes(T.pslots[p]);
            c.slab = (unsigned)s;
            c.row0 = u.sb0 * kStmRS;
            c.flags = pf;
            c.half = (unsigned char)q;
            c.sp = (unsigned char)u.sp;
            cmds.push_back(c);
          }
        }
      if (cmds.size() == first) {  // nothing in range: header-only stage closes the unit
        StmCmd c{};
        c.row0 = u.sb0 * kStmRS;
        c.flags = pf;
        c.sp = (unsigned char)u.sp;
        cmds.push_back(c);
      }
      cmds.back().flags |= STM_END;
    }
  }
  coff[G] = (long long)cmds.size();
  S.cmds = dalloc<StmCmd>(h, std::max<size_t>(cmds.size(), 1));
  S.coff = dalloc<long long>(h, G + 1);
  h2d(h, S.cmds, cmds.data(), cmds.size());
  h2d(h, S.coff, coff.data(), G + 1);
  S.G = G;
  S.splits = splits;
  S.ncmd = (long long)cmds.size();
  dbg("stream sched mat=%d pair=%d units=%zu tiled=%lld splits=%d G=%d cmds=%zu", mat, pair,
      all.size(), ntiled, splits, G, cmds.size());
}

void build_stream(scs_handle* h, int mat) {
  const Csr& M = mat == 0 ? h->A : h->At;
  const long long rows = M.rows, cols = mat == 0 ? h->n : h->m;
  const long long nz = read_dev(h, M.rp + rows);
  Stm& F = h->sF[mat];
  F.rows = rows;
  F.cols = cols;
  // slab width: 4096 columns, narrowed (/4, down to 256) when dense rows
  // make warp sections deeper than k_stm_pin handles (> 0.1% flagged)
  const bool wforced = getenv("SCS_STREAM_W") != nullptr;
  long long W = std::min<long long>(kStmMaxW, std::max<long long>(32, env_ll("SCS_STREAM_W", 4096)));  // >= 32: padding gathers column = lane
  F.cap = (int)(env_ll("SCS_STREAM_CAP", 0) & ~15LL);
  const int min_cap = (int)stm_piece_bytes(32 * kStmWarps);
  if (F.cap > 0 && F.cap < min_cap) F.cap = (min_cap + 15) & ~15;
  F.NB = (int)((rows + kStmRS - 1) / kStmRS);
  std::vector<long long> rp_h(rows + 1);
  d2h(h, rp_h.data(), M.rp, rows + 1);
  CK(cudaStreamSynchronize(h->st));
  if (!wforced && nz > 0 && env_ll("SCS_STREAM_PREDICT", 1)) {
    // expected section depth in the densest slab (column counts from the
    // other CSR's row pointers): narrow the slab up front where sub-blocks
    // would exceed the pin depth, instead of building and rebuilding (the
    // build below still narrows further if sections get flagged)
    const Csr& O = mat == 0 ? h->At : h->A;
    std::vector<long long> orp(cols + 1);
    d2h(h, orp.data(), O.rp, cols + 1);
    CK(cudaStreamSynchronize(h->st));
    for (; W > 256; W /= 4) {
      long long smax = 0;
      for (long long c0 = 0; c0 < cols; c0 += W) smax = std::max(smax, orp[std::min(cols, c0 + W)] - orp[c0]);
      const double frac = (double)smax / (double)nz;
      long long deep = 0, nsb = 0;
      for (long long r0 = 0; r0 < rows; r0 += kStmRS) {
        const long long e = rp_h[std::min(rows, r0 + kStmRS)] - rp_h[r0];
        nsb += e > 0;
        deep += (double)e / kStmWarps * frac / 32.0 > 96.0;
      }
      if (deep * 1000 <= nsb) break;
    }
  }
  long long ntile = 0, nsec = 0;
  int *rowid = nullptr, *perm = nullptr, *sec = nullptr, *slot = nullptr;
  unsigned char* hown = nullptr;
  std::vector<unsigned short> D;
  for (;;) {
  F.W = (int)W;
  F.S = (int)((cols + F.W - 1) / F.W);
  ntile = (long long)F.NB * F.S;
  nsec = ntile * kStmWarps;
  if (nsec >= (1LL << 31) - 1 || nz >= (1LL << 31) - 1 || nz == 0)
    throw Fail{SCS_EINVAL, "streamed layout: too many sections or nonzeros"};
  // 1. entries by (warp section, owning lane, rotated gather bank)
  rowid = dalloc<int>(h, nz);
  unsigned long long* key = dalloc<unsigned long long>(h, nz);
  unsigned long long* skey = dalloc<unsigned long long>(h, nz);
  int* perm_in = dalloc<int>(h, nz);
  perm = dalloc<int>(h, nz);
  k_expand_rows<<<elem_grid(h, rows * 32), kBlock, 0, h->st>>>(M.rp, rows, rowid);
  k_stm_keys<<<elem_grid(h, nz), kBlock, 0, h->st>>>(rowid, M.ci, nz, F.W, F.S, key);
  k_iota<<<elem_grid(h, nz), kBlock, 0, h->st>>>(perm_in, nz);
  int bits = 1;
  while ((1LL << bits) < nsec) ++bits;
  {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const unsigned long long*)key, skey,
                                       (const int*)perm_in, perm, (int)nz, 0, bits + 12, h->st));
    void* tmp = dalloc<char>(h, tb);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, (const unsigned long long*)key, skey,
                                       (const int*)perm_in, perm, (int)nz, 0, bits + 12, h->st));
    CK(cudaStreamSynchronize(h->st));
    dfree(h, tmp);
  }
  dfree(h, key);
  dfree(h, perm_in);
  dbg("stream mat=%d: sorted", mat);
  // 2. sections, slots (pinned / overflow) and depths
  sec = dalloc<int>(h, nz);
  k_stm_sec<<<elem_grid(h, nz), kBlock, 0, h->st>>>(skey, nz, sec);
  long long* sec_ptr = dalloc<long long>(h, nsec + 1);
  k_rowptr<<<elem_grid(h, nsec + 1), kBlock, 0, h->st>>>(sec, nz, nsec, sec_ptr);
  slot = dalloc<int>(h, nz);
  unsigned short* depth = dalloc<unsigned short>(h, nsec);
  hown = dalloc<unsigned char>(h, nsec * 32);
  k_stm_pin<<<elem_grid(h, nsec), kBlock, 0, h->st>>>(sec_ptr, nsec, skey, perm, slot, depth, hown);
  CK(cudaGetLastError());
  D.assign(nsec, 0);
  d2h(h, D.data(), depth, nsec);
  CK(cudaStreamSynchronize(h->st));
  dbg("stream mat=%d: pinned", mat);
  dfree(h, depth);
  dfree(h, sec_ptr);
  dfree(h, skey);
  long long nbad = 0, nne = 0;
  for (long long q = 0; q < nsec; ++q) {
    nbad += D[q] == 0xffff;
    nne += D[q] != 0;
  }
  dbg("stream pin mat=%d W=%d sections=%lld flagged=%lld", mat, F.W, nne, nbad);
  if (wforced || W <= 256 || nbad * 1000 <= nne) break;
  for (void* p : {(void*)rowid, (void*)perm, (void*)sec, (void*)slot, (void*)hown}) dfree(h, p);
  W /= 4;
  }
  if (F.cap <= 0) {
    // default piece cap: three stages beside the accumulators and two slab
    // buffers of an NV = 1 pass, so that a piece is a whole tile (~42 KB at
    // config 5): measured at C5, whole-tile pieces beat deeper rings of
    // smaller pieces (the per-piece synchronisation of 16 consumer warps
    // costs more than the extra bytes in flight gain), and single sub-block
    // units (32 KB of accumulators) beat slab-sharing pairs (64 KB), whose
    // stages would have to be half as large
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
    const long long avail = (long long)optin - 1024 - (h->stm_pair ? 2 : 1) * kStmRS * 8LL -
                            2LL * F.W * 8 - kStmMaxStages * (2 * 8 + 16);
    const long long nst = env_ll("SCS_STREAM_STAGES", 3);
    F.cap = (int)(std::min<long long>(65536, std::max<long long>(min_cap, avail / nst)) & ~15LL);
    if (F.cap < min_cap) F.cap = (min_cap + 15) & ~15;
  }
  dbg("stream piece cap mat=%d: %d bytes", mat, F.cap);
  // 5. host: tiled sub-blocks, pieces, blob offsets
  StmTiles T;
  T.NB = F.NB;
  T.S = F.S;
  T.tiled.assign(F.NB, 1);
  T.pf.assign(ntile, -1);
  T.np.assign(ntile, 0);
  T.slots.assign(ntile, 0);
  T.nnz_sb.assign(F.NB, 0);
  const long long min_avg = env_ll("SCS_STREAM_MIN", 768);
  for (long long sb = 0; sb < F.NB; ++sb) {
    const long long r0 = sb * kStmRS, r1 = std::min(rows, r0 + kStmRS);
    T.nnz_sb[sb] = rp_h[r1] - rp_h[r0];
    long long sl = 0, nt = 0;
    bool bad = false;
    for (long long s = 0; s < F.S; ++s) {
      long long a = 0;
      for (int w = 0; w < kStmWarps; ++w) {
        const unsigned short d = D[(sb * F.S + s) * kStmWarps + w];
        if (d == 0xffff) bad = true;
        else a += 32LL * d;
      }
      T.slots[sb * F.S + s] = a;
      sl += a;
      nt += a > 0;
    }
    // CSR units only for short rows (the consumers run them at 4 lanes per row)
    T.tiled[sb] = !bad && (nt == 0 || sl >= min_avg * nt || T.nnz_sb[sb] > 16 * (r1 - r0)) ? 1 : 0;
  }
  // pieces: consecutive step ranges [s_j, s_j+1) of all sections of a tile,
  // each grown greedily up to `cap` bytes, so the ring's stages carry full
  // pieces (the bytes in flight per SM set the achievable DRAM rate)
  std::vector<unsigned short> pstep0, pwsec;
  std::vector<long long> ptile;  // tile of every piece
  long long npiece = 0;
  unsigned long long bytes = 0;
  for (long long t = 0; t < ntile; ++t) {
    if (!T.tiled[t / F.S] || T.slots[t] == 0) continue;
    const unsigned short* d = &D[t * kStmWarps];
    int maxd = 0;
    for (int w = 0; w < kStmWarps; ++w) maxd = std::max<int>(maxd, d[w]);
    T.pf[t] = npiece;
    int np = 0;
    for (int s0 = 0; s0 < maxd;) {
      long long cnt = 0;
      int e = s0;
      for (;;) {  // at least one step (a step of every section fits: cap >= min_cap)
        long long add = 0;
        for (int w = 0; w < kStmWarps; ++w) add += d[w] > e;
        if (e > s0 && stm_piece_bytes(32ULL * (cnt + add)) > (unsigned long long)F.cap) break;
        cnt += add;
        if (++e >= maxd) break;
      }
      unsigned short acc = 0;
      pwsec.push_back(0);
      for (int w = 0; w < kStmWarps; ++w) {
        const int st = std::max(0, std::min<int>(d[w], e) - s0);
        acc = (unsigned short)(acc + st);
        pwsec.push_back(acc);
      }
      const unsigned ns = 32u * acc;
      T.poff.push_back(bytes);
      ptile.push_back(t);
      pstep0.push_back((unsigned short)s0);
      T.pslots.push_back(ns);
      bytes += stm_piece_bytes(ns);
      ++npiece;
      ++np;
      s0 = e;
    }
    T.np[t] = np;
  }
  dbg("stream mat=%d: piece table (%lld pieces)", mat, npiece);
  // 6. device blob
  unsigned char* blob = dalloc<unsigned char>(h, std::max<unsigned long long>(bytes, 16));
  long long* d_pf = dalloc<long long>(h, ntile);
  unsigned short* d_ps0 = dalloc<unsigned short>(h, std::max<long long>(npiece, 1));
  int* d_np = dalloc<int>(h, ntile);
  unsigned long long* d_poff = dalloc<unsigned long long>(h, npiece);
  unsigned* d_pslots = dalloc<unsigned>(h, npiece);
  unsigned short* d_pwsec = dalloc<unsigned short>(h, pwsec.size());
  h2d(h, d_pf, T.pf.data(), ntile);
  h2d(h, d_ps0, pstep0.data(), npiece);
  h2d(h, d_np, T.np.data(), ntile);
  h2d(h, d_poff, T.poff.data(), npiece);
  h2d(h, d_pslots, T.pslots.data(), npiece);
  h2d(h, d_pwsec, pwsec.data(), pwsec.size());
  if (npiece) {
    long long* d_ptile = dalloc<long long>(h, npiece);
    h2d(h, d_ptile, ptile.data(), npiece);
    k_stm_init<<<elem_grid(h, npiece * 32), kBlock, 0, h->st>>>(blob, d_poff, d_pslots, d_pwsec,
                                                                d_ptile, hown, npiece);
    k_stm_scatter<<<elem_grid(h, nz), kBlock, 0, h->st>>>(sec, slot, nz, perm, rowid, M.ci, M.v, d_pf,
                                                          d_ps0, d_np, d_poff, d_pslots, d_pwsec, F.W, blob);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->st));
    dfree(h, d_ptile);
  }
  CK(cudaStreamSynchronize(h->st));
  for (void* p : {(void*)d_pf, (void*)d_ps0, (void*)d_np, (void*)d_poff, (void*)d_pslots, (void*)d_pwsec,
                  (void*)sec, (void*)slot, (void*)perm, (void*)rowid, (void*)hown})
    dfree(h, p);
  F.blob = blob;
  h->stm_bytes[mat] = bytes;
  long long ncsr = 0;
  for (long long sb = 0; sb < F.NB; ++sb) ncsr += !T.tiled[sb];
  dbg("stream layout mat=%d rows=%lld cols=%lld nnz=%lld W=%d S=%d NB=%d csr_sb=%lld pieces=%lld "
      "bytes=%llu (%.2f B/nnz)", mat, rows, cols, nz, F.W, F.S, F.NB, ncsr, npiece, bytes,
      (double)bytes / (double)nz);
  for (int pair = 0; pair < 2; ++pair)
    build_stm_sched(h, mat, pair, T, 0, F.NB, h->ssch[mat][pair], h->sms);
  // row-sharded A^T passes: also one schedule per row chunk, so the all-
  // reduce of chunk c overlaps the SpMV of chunk c + 1 (at_pass); a few SMs
  // stay free for the NCCL kernels
  if (mat == 1 && h->sharded && h->at_chunks > 1) {
    const int C = h->at_chunks;
    const int G = std::max(1, h->sms - (int)env_ll("SCS_AT_FREE_SMS", 8));
    for (int c = 0; c < C; ++c) {
      const long long lo = F.NB * c / C, hi = F.NB * (c + 1) / C;
      h->at_row[c] = std::min(F.rows, lo * kStmRS);
      for (int pair = 0; pair < 2; ++pair) build_stm_sched(h, mat, pair, T, lo, hi, h->at_sch[c][pair], G);
    }
    h->at_row[C] = F.rows;
  }
}

__global__ void k_hash_fill(double* x, long long n, unsigned seed) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n; i += nt) {
    unsigned long long z = (unsigned long long)i * 0x9E3779B97F4A7C15ULL + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    x[i] = (double)((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

// SCS_STREAM_CHECK=1: streamed products against the CSR kernel for every
// (NV, STRIDE) shape the iteration uses; max |difference| to stderr.
void stm_selfcheck(scs_handle* h) {
  for (int mat = 0; mat < 2; ++mat) {
    const long long rows = mat == 0 ? h->m : h->n, cols = mat == 0 ? h->n : h->m;
    double* x = dalloc<double>(h, 2 * cols);
    double* o1 = dalloc<double>(h, 2 * rows);
    double* o2 = dalloc<double>(h, 2 * rows);
    k_hash_fill<<<elem_grid(h, 2 * cols), kBlock, 0, h->st>>>(x, 2 * cols, 17u + mat);
    auto cmp = [&](const char* what, long long len) {
      std::vector<double> a(len), b(len);
      d2h(h, a.data(), o1, len);
      d2h(h, b.data(), o2, len);
      CK(cudaStreamSynchronize(h->st));
      double mx = 0.0, sc = 0.0;
      long long arg = -1;
      for (long long i = 0; i < len; ++i) {
        const double d = std::fabs(a[i] - b[i]);
        if (!(d <= mx)) { mx = d; arg = i; }
        sc = std::max(sc, std::fabs(b[i]));
      }
      fprintf(stderr, "[scs] stream check mat=%d %s max|diff|=%.3e at %lld (scale %.3e)\n", mat, what,
              mx, arg, sc);
    };
    {
      EpiPlainN<1, 1> e{};
      e.V = h->V; e.xb = x; e.out = o1;
      launch_stream<1, 1>(h, mat, e);
      e.out = o2;
      launch_spmv(h, mat == 0 ? h->A : h->At, mat == 0 ? h->LA : h->LAt, e);
      cmp("nv1s1", rows);
    }
    {
      EpiPlainN<1, 2> e{};
      e.V = h->V; e.xb = x; e.out = o1;
      launch_stream<1, 2>(h, mat, e);
      e.out = o2;
      launch_spmv(h, mat == 0 ? h->A : h->At, mat == 0 ? h->LA : h->LAt, e);
      cmp("nv1s2", rows);
    }
    {
      EpiPlainN<2, 2> e{};
      e.V = h->V; e.xb = x; e.out = o1;
      launch_stream<2, 2>(h, mat, e);
      e.out = o2;
      launch_spmv(h, mat == 0 ? h->A : h->At, mat == 0 ? h->LA : h->LAt, e);
      cmp("nv2s2", 2 * rows);
    }
    dfree(h, x);
    dfree(h, o1);
    dfree(h, o2);
  }
}

// Streamed tiles for large matrices (SCS_STREAM=0 off, 1 force on).
void setup_stream(scs_handle* h) {
  const long long force = env_ll("SCS_STREAM", -1);
  h->stm_pair = env_ll("SCS_STREAM_PAIR", 0) != 0;
  // (r02) from 4e6 nonzeros (dense tiles, tools/r02_stream_vs_csr.py --small:
  // 2.7e6 181 vs 168 us per iteration for the CSR kernel, 5.3e6 218 vs 246,
  // 1.05e7 291 vs 433; r01: from 2e7)
  const bool gate = force > 0 || (force < 0 && h->nnz >= env_ll("SCS_STREAM_NNZ_MIN", 4000000LL));
  // (r02) per matrix: the streamed format pays a slab load (W columns of
  // the gathered vector) and a piece header per tile, so it only wins when
  // the average tile holds enough entries -- measured at 2.1e7 nonzeros:
  // 3428 entries per tile 1.6x faster than the CSR kernel, 175 / 88 / 22
  // entries per tile 2-3x slower, crossover near 1000 (800: 15% slower,
  // 1200: 13% faster; tools/r02_stream_vs_csr.py); config 5: 1671, config
  // 3: 16,300.  Below the threshold the matrix stays CSR.
  const long long tile_min = env_ll("SCS_STREAM_TILE_MIN", 1000);
  bool want[2] = {false, false};
  for (int mat = 0; mat < 2 && gate && h->nnz > 0; ++mat) {
    want[mat] = true;
    if (force > 0) continue;
    const long long rows = mat == 0 ? h->m : h->n, cols = mat == 0 ? h->n : h->m;
    const double tiles = (double)((rows + kStmRS - 1) / kStmRS) * (double)((cols + kStmMaxW - 1) / kStmMaxW);
    if ((double)h->nnz < (double)tile_min * tiles) {
      dbg("stream mat=%d: %.0f entries per tile < %lld, CSR kernel", mat, (double)h->nnz / tiles, tile_min);
      want[mat] = false;
    }
    // ... and enough tiles to spread over the persistent CTAs (units x slab
    // ranges): bench config s1e7 (1e7 nonzeros in 25 x 3 tiles) ran at half
    // the CSR kernel's rate streamed; 124 tiles 8% slower, 434 tiles 12% faster
    else if (tiles < (double)env_ll("SCS_STREAM_TILES_MIN", 2LL * h->sms)) {
      dbg("stream mat=%d: %.0f tiles < 2 per SM, CSR kernel", mat, tiles);
      want[mat] = false;
    }
  }
  // Row-sharded: the A^T pass's collectives follow its format (chunked
  // all-reduces when streamed), so every rank makes the same choice -- a
  // matrix is streamed only where every rank's shard wants it.
  if (h->sharded) {
    double w[2] = {want[0] ? 1.0 : 0.0, want[1] ? 1.0 : 0.0};
    double* d = dalloc<double>(h, 2);
    h2d(h, d, w, 2);
    allreduce(h, d, 2);
    CK(cudaMemcpyAsync(w, d, sizeof(w), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    dfree(h, d);
    for (int mat = 0; mat < 2; ++mat) want[mat] = w[mat] >= (double)h->world - 0.5;
  }
  if (!want[0] && !want[1]) return;
  h->at_chunks = h->sharded ? (int)std::max<long long>(1, std::min<long long>(
                                    scs_handle::kMaxChunks, env_ll("SCS_AT_CHUNKS", 2)))
                             : 1;
  size_t need = 0;
  for (int mat = 0; mat < 2; ++mat) {
    if (!want[mat]) continue;
    build_stream(h, mat);
    h->stm_m[mat] = true;
    for (int pair = 0; pair < 2; ++pair) {
      int sp = h->ssch[mat][pair].splits;
      if (mat == 1)
        for (int c = 0; c < h->at_chunks && h->at_chunks > 1; ++c) sp = std::max(sp, h->at_sch[c][pair].splits);
      if (sp > 1) need = std::max<size_t>(need, (size_t)sp * h->sF[mat].rows * 2);
    }
  }
  if (h->at_chunks > 1) {
    CK(cudaStreamCreateWithFlags(&h->st_comm, cudaStreamNonBlocking));
    for (int c = 0; c < h->at_chunks; ++c) CK(cudaEventCreateWithFlags(&h->ev_chunk[c], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming));
  }
  if (need) h->Pstm = dalloc<double>(h, need);
  if (env_ll("SCS_STREAM_CHECK", 0)) stm_selfcheck(h);
}

__global__ void k_pcg_diag(const double* colsq, long long n, double* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long j = tid; j < n; j += nt) out[j] = 1.0 / (1.0 + colsq[j]);
}

// Opt-in Jacobi PCG: M^-1 = 1 / (1 + ||A_hat e_j||^2) from the equilibrated
// CSR(A^T) (column sums all-reduced when rows are sharded).
void setup_pcg(scs_handle* h) {
  if (!(h->set.fast & SCS_FAST_PCG)) return;
  const long long n = h->n;
  h->Minv = dalloc<double>(h, n);
  k_row_sumsq<<<elem_grid(h, n * 32), kBlock, 0, h->st>>>(h->At, h->tmp_n);
  allreduce(h, h->tmp_n, n);
  k_pcg_diag<<<elem_grid(h, n), kBlock, 0, h->st>>>(h->tmp_n, n, h->Minv);
  CK(cudaStreamSynchronize(h->st));
  h->V.Minv = h->Minv;
}

// Skewed rows (SURVEY §7 hard part 1): a CSR kernel with L lanes per row
// runs a row of R nonzeros in ~R/(4L) dependent load rounds, so one dense
// row (config 4: the budget row and the factor rows hold all 1e5 assets)
// costs milliseconds while the average row is tiny.  When the longest row
// exceeds 128 x the kernel's design point (8 nonzeros per lane), rows are
// cut into pieces of at most 32 L entries -- a refined row pointer into the
// same (ci, v) arrays, no data movement -- the pass writes raw piece
// products and the epilogue kernel (k_rows with `seg`) sums each row's
// pieces in order before running the epilogue.
void setup_split(scs_handle* h) {
  const char* env = getenv("SCS_SPLIT");
  const int force = env ? atoi(env) : -1;  // 0 off, 1 on (any long row), unset: heuristic
  if (force == 0 || h->nnz == 0) return;
  size_t need = 0;
  for (int mat = 0; mat < 2; ++mat) {
    if (h->stm_m[mat]) continue;
    const Csr& M = mat == 0 ? h->A : h->At;
    const long long rows = M.rows;
    std::vector<long long> rp(rows + 1);
    CK(cudaMemcpy(rp.data(), M.rp, (rows + 1) * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (long long i = 0; i < rows; ++i) mx = std::max(mx, rp[i + 1] - rp[i]);
    const int L = mat == 0 ? h->LA : h->LAt;
    const long long cap = force == 1 ? std::max<long long>(8, 4LL * L) : 32LL * L;
    if (mx <= (force == 1 ? cap : 128LL * 8 * L)) continue;
    std::vector<long long> seg(rows + 1), vrp;
    vrp.reserve(rows + h->nnz / cap + 2);
    for (long long i = 0; i < rows; ++i) {
      seg[i] = (long long)vrp.size();
      long long k = rp[i];
      do {
        vrp.push_back(k);
        k += cap;
      } while (k < rp[i + 1]);
    }
    seg[rows] = (long long)vrp.size();
    vrp.push_back(rp[rows]);
    std::vector<long long> lr;
    for (long long i = 0; i < rows; ++i)
      if (seg[i + 1] - seg[i] > kLongSeg) lr.push_back(i);
    if (!lr.empty()) {
      h->long_rows[mat] = dalloc<long long>(h, lr.size());
      h2d(h, h->long_rows[mat], lr.data(), lr.size());
      h->n_long[mat] = (long long)lr.size();
    }
    const long long V = (long long)vrp.size() - 1;
    long long* dv = dalloc<long long>(h, V + 1);
    long long* ds = dalloc<long long>(h, rows + 1);
    h2d(h, dv, vrp.data(), V + 1);
    h2d(h, ds, seg.data(), rows + 1);
    CK(cudaStreamSynchronize(h->st));
    h->Asp[mat] = Csr{dv, M.ci, M.v, V};
    h->seg[mat] = ds;
    h->Lsp[mat] = pick_lanes(h->nnz, V);
    h->split_m[mat] = true;
    need = std::max<size_t>(need, 2 * (size_t)V);
    dbg("split: mat=%d rows=%lld longest=%lld pieces=%lld cap=%lld L=%d", mat, rows, mx, V, cap,
        h->Lsp[mat]);
  }
  if (need) h->Psplit = dalloc<double>(h, need);
}

// A pass over the local rows.  Row-sharded: its (y-part) totals are
// all-reduced and finished by k_finish.
template <class Epi>
void a_pass(scs_handle* h, Epi epi) {
  if (gated_off(h, epi.rgate)) return;
  epi.defer = (h->sharded && Epi::NR > 0) ? 1 : 0;
  launch_mat(h, 0, epi);
  if (epi.defer) {
    allreduce(h, h->V.dred, Epi::NR);
    k_finish<Epi><<<1, 32, 0, h->st>>>(epi);
    h->launches++;
  }
}

// A^T pass.  Row-sharded: raw partial products of the local rows, one
// all-reduce of NV n-vectors, then the epilogue on the reduced products
// (its reductions are over replicated x-space data: no further all-reduce).
template <class Epi>
void at_pass(scs_handle* h, Epi epi) {
  if (gated_off(h, epi.rgate)) return;
  epi.defer = 0;
  if (!h->sharded) {
    launch_mat(h, 1, epi);
    return;
  }
  const long long n = h->n;
  EpiRaw<Epi> raw{};
  static_cast<Epi&>(raw) = epi;
  raw.T = h->Traw;
  if (h->at_chunks > 1 && h->stm_m[1] && ((uintptr_t)raw.xb & 15) == 0) {
    // chunk c's raw products all-reduced on st_comm while chunk c + 1 runs
    for (int c = 0; c < h->at_chunks; ++c) {
      launch_stream<EpiRaw<Epi>::NV, EpiRaw<Epi>::STRIDE, EpiRaw<Epi>>(h, 1, raw, c);
      CK(cudaEventRecord(h->ev_chunk[c], h->st));
      CK(cudaStreamWaitEvent(h->st_comm, h->ev_chunk[c], 0));
      const long long a = h->at_row[c], b = h->at_row[c + 1];
      if (b > a) h->comm->allreduce(h->st_comm, h->Traw + a * Epi::NV, (size_t)(b - a) * Epi::NV);
    }
    CK(cudaEventRecord(h->ev_comm, h->st_comm));
    CK(cudaStreamWaitEvent(h->st, h->ev_comm, 0));
  } else {
    launch_mat(h, 1, raw);
    allreduce(h, h->Traw, (size_t)n * Epi::NV);
  }
  k_rows<Epi><<<elem_grid(h, n), kBlock, 0, h->st>>>(h->Traw, n, 1, epi);
  h->launches++;
}

// Elementwise epilogue over an m-vector of A products (split CSR path);
// its y-part totals are all-reduced when rows are sharded.
template <class Epi>
void y_rows(scs_handle* h, const double* T, Epi epi) {
  if (gated_off(h, epi.rgate)) return;
  epi.defer = (h->sharded && Epi::NR > 0) ? 1 : 0;
  k_rows<Epi><<<elem_grid(h, h->m), kBlock, 0, h->st>>>(T, h->m, 1, epi);
  h->launches++;
  if (epi.defer) {
    allreduce(h, h->V.dred, Epi::NR);
    k_finish<Epi><<<1, 32, 0, h->st>>>(epi);
    h->launches++;
  }
}

// final A pass of solve_kkt: z_y = rhs_y + A x (embedding.py:113)
void a_final(scs_handle* h, const Vec& V, double* zy_out, int setup) {
  const bool recur = !setup && (h->set.fast & SCS_FAST_RECURRENCE);
  if (!h->stm_m[0] || recur) {
    EpiAxPlain ax{};
    ax.V = V;
    ax.xb = V.x;
    ax.gate = recur ? h->recur_refresh : 0;
    launch_mat(h, 0, ax);
    EpiZy ez{};
    ez.V = V;
    ez.zy_out = zy_out;
    ez.setup = setup;
    y_rows(h, V.Axw, ez);
    return;
  }
  EpiAFinal ef{};
  ef.V = V;
  ef.xb = V.x;
  ef.zy_out = zy_out;
  ef.setup = setup;
  a_pass(h, ef);
}

// ---------------------------------------------------------------------------
// cone layout of this shard: rows [row_lo, row_lo + m) of the global cone
// ---------------------------------------------------------------------------
void build_cones(scs_handle* h, const scs_problem* P) {
  const long long lo = h->row_lo, hi = h->row_lo + h->m;
  const std::vector<long long>& B = h->bounds;
  auto cut = [&](long long a, long long b) {  // block [a, b) split by a shard bound
    for (size_t k = 1; k + 1 < B.size(); ++k)
      if (B[k] > a && B[k] < b) return true;
    return false;
  };
  std::vector<long long> ssoc_off;
  std::vector<int> ssoc_len;
  std::vector<long long> bsoc_off, bsoc_len;
  std::vector<int> bsoc_chunk_lo, bsoc_gid;
  std::vector<long long> chunk_off;
  std::vector<int> chunk_len, chunk_cone;
  std::vector<long long> psd_off;
  std::vector<int> psd_side;
  std::vector<long long> seg_off, seg_len, seg_glen;
  std::vector<int> seg_gid;
  // zero and nonneg rows: the shard's share of [0, z) and [z, z + l)
  const long long z = P->z, l = P->l;
  h->K.z = std::max(0LL, std::min(z, hi) - lo);
  h->K.l = std::max(0LL, std::min(z + l, hi) - std::max(z, lo));
  if (h->K.z < 0 || h->K.l < 0) throw Fail{SCS_EINVAL, "internal: bad zero/nonneg share"};
  long long off = z + l;
  int ng = 0, sg = 0;
  for (long long i = 0; i < P->nq; ++i) {  // cones.py:134-136
    const long long d = P->q[i];
    if (d < 1) throw Fail{SCS_EINVAL, "second-order cone dims must be >= 1"};
    const bool big = d > kSmallSoc || cut(off, off + d);
    const long long a = std::max(off, lo), b = std::min(off + d, hi);
    if (b > a) {
      seg_off.push_back(a - lo);
      seg_len.push_back(b - a);
      seg_gid.push_back(sg);
      if (!big) {
        ssoc_off.push_back(off - lo);
        ssoc_len.push_back((int)d);
      } else {
        bsoc_off.push_back(off - lo);  // negative when the head lives on another shard
        bsoc_len.push_back(d);
        bsoc_gid.push_back(ng);
        bsoc_chunk_lo.push_back((int)chunk_off.size());
        for (long long e = a; e < b; e += kChunk) {
          chunk_off.push_back(e - lo);
          chunk_len.push_back((int)std::min<long long>(kChunk, b - e));
          chunk_cone.push_back((int)bsoc_off.size() - 1);
        }
      }
    }
    seg_glen.push_back(d);
    ++sg;
    if (big) ++ng;
    off += d;
  }
  bsoc_chunk_lo.push_back((int)chunk_off.size());
  h->K.n_big_global = ng;
  long long psd_lo = -1, psd_hi = -1;
  int max_side = 0;
  for (long long i = 0; i < P->ns; ++i) {  // cones.py:137-139
    const long long k = P->s[i];
    if (k < 1) throw Fail{SCS_EINVAL, "PSD side lengths must be >= 1"};
    const long long d = k * (k + 1) / 2;
    if (cut(off, off + d)) throw Fail{SCS_EINVAL, "a shard bound cuts a PSD block"};
    if (off >= lo && off + d <= hi) {
      psd_off.push_back(off - lo);
      psd_side.push_back((int)k);
      max_side = std::max<int>(max_side, (int)k);
      if (psd_lo < 0) psd_lo = off - lo;
      psd_hi = off + d - lo;
      seg_off.push_back(off - lo);
      seg_len.push_back(d);
      seg_gid.push_back(sg);
    }
    seg_glen.push_back(d);
    ++sg;
    off += d;
  }
  h->K.psd_lo = psd_lo < 0 ? 0 : psd_lo;
  h->K.psd_hi = psd_hi < 0 ? 0 : psd_hi;
  long long n_exp = 0, exp_lo = -1;
  for (long long i = 0; i < P->ep; ++i) {
    if (cut(off, off + 3)) throw Fail{SCS_EINVAL, "a shard bound cuts an exponential cone"};
    if (off >= lo && off + 3 <= hi) {
      if (exp_lo < 0) exp_lo = off - lo;
      ++n_exp;
      seg_off.push_back(off - lo);
      seg_len.push_back(3);
      seg_gid.push_back(sg);
    }
    seg_glen.push_back(3);
    ++sg;
    off += 3;
  }
  h->K.exp_lo = exp_lo < 0 ? 0 : exp_lo;
  h->K.n_exp = n_exp;
  if (off != h->m_glob)
    throw Fail{SCS_EINVAL, "cone dimension " + std::to_string(off) + " does not match row count " +
                               std::to_string(h->m_glob)};
  auto up_ll = [&](const std::vector<long long>& v) {
    long long* d = dalloc<long long>(h, v.size());
    h2d(h, d, v.data(), v.size());
    return d;
  };
  auto up_i = [&](const std::vector<int>& v) {
    int* d = dalloc<int>(h, v.size());
    h2d(h, d, v.data(), v.size());
    return d;
  };
  h->K.n_ssoc = (int)ssoc_off.size();
  h->K.ssoc_off = up_ll(ssoc_off);
  h->K.ssoc_len = up_i(ssoc_len);
  h->K.n_bsoc = (int)bsoc_off.size();
  h->K.bsoc_off = up_ll(bsoc_off);
  h->K.bsoc_len = up_ll(bsoc_len);
  h->K.bsoc_gid = up_i(bsoc_gid);
  h->K.bsoc_chunk_lo = up_i(bsoc_chunk_lo);
  h->K.n_chunk = (int)chunk_off.size();
  h->K.chunk_off = up_ll(chunk_off);
  h->K.chunk_len = up_i(chunk_len);
  h->K.chunk_cone = up_i(chunk_cone);
  h->K.n_psd = (int)psd_off.size();
  h->K.psd_off = up_ll(psd_off);
  h->K.psd_side = up_i(psd_side);
  h->K.max_side = max_side;
  h->cone_red_len = 3 + 2 * ng;
  // equilibration segments: every non-singleton block (scaling.py:62-71)
  h->nseg = (int)seg_off.size();
  h->nseg_g = sg;
  h->seg_off = up_ll(seg_off);
  h->seg_len = up_ll(seg_len);
  h->seg_gid = up_i(seg_gid);
  h->seg_glen = up_ll(seg_glen);
  h->seg_sum = dalloc<double>(h, std::max(sg, 1));
  h->seg_mean = dalloc<double>(h, std::max(sg, 1));
  // PSD workspace: shared memory up to ~200 KB, else global scratch
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  const size_t budget = (size_t)std::max(0, optin - 12 * 1024);  // minus static smem
  int side = 0;
  while ((size_t)2 * (side + 1) * (side + 1) * sizeof(double) <= budget) ++side;
  h->smem_side = std::min(side, 255);
  if (const char* e = getenv("SCS_PSD_WARP")) h->warp_side = atoi(e) ? kWarpPsd : 0;
  const int s_used = max_side > h->warp_side ? std::min(max_side, h->smem_side) : 0;
  // CTA-per-block region for large blocks; per-warp regions for small ones
  h->cone_smem = (size_t)2 * s_used * s_used * sizeof(double);
  h->n_psd_small = 0;
  {
    std::vector<int> small;
    for (size_t b = 0; b < psd_side.size(); ++b)
      if (psd_side[b] <= h->warp_side) small.push_back((int)b);
    std::stable_sort(small.begin(), small.end(),
                     [&](int a, int b) { return psd_side[a] > psd_side[b]; });
    h->n_psd_small = (int)small.size();
    if (!small.empty()) h->psd_small_list = up_i(small);
  }
  // blocks beyond the shared-memory side: M, V (and the rotation-pair
  // arrays when > 128 pairs) in global scratch, one region per block
  {
    std::vector<long long> goff(psd_side.size(), -1);
    long long tot = 0;
    for (size_t b = 0; b < psd_side.size(); ++b) {
      const long long k = psd_side[b];
      if (k <= h->smem_side || k <= h->warp_side) continue;
      goff[b] = tot;
      tot += 2 * k * k + 5 * ((k + 1) / 2) + 8;
    }
    if (tot) h->psd_scratch = dalloc<double>(h, tot);
    if (!goff.empty()) h->K.psd_goff = up_ll(goff);
  }
  // those blocks go to the cooperative-grid Jacobi (SCS_PSD_GRID=0: one CTA
  // each in k_cone_apply, the r01 path) while its pair table fits in smem
  {
    bool use = true;
    if (const char* e = getenv("SCS_PSD_GRID")) use = atoi(e) != 0;
    // emulated group: several shards share this GPU, and two partly resident
    // cooperative grids could wait on each other's SMs -- one CTA per block
    if (h->comm && dynamic_cast<EmuComm*>(h->comm)) use = false;
    std::vector<int> big;
    int kmax = 0;
    if (use) {
      h->psd_grid_max = h->smem_side;
      while (psd_grid_pair_bytes(h->psd_grid_max + 1) <= budget) ++h->psd_grid_max;
    }
    for (size_t b = 0; b < psd_side.size() && use; ++b) {
      const int k = psd_side[b];
      if (k <= h->smem_side || k <= h->warp_side || k > h->psd_grid_max) continue;
      big.push_back((int)b);
      kmax = std::max(kmax, k);
    }
    if (!big.empty()) {
      h->n_psd_grid = (int)big.size();
      h->psd_grid_list = up_i(big);
      h->psd_grid_smem = std::max(kPsdTileSmem, psd_grid_pair_bytes(kmax));
      if ((size_t)smem_optin(h, (const void*)k_psd_grid) < h->psd_grid_smem)
        throw Fail{SCS_ECUDA, "k_psd_grid: shared memory budget exceeded"};
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_psd_grid, kBlock,
                                                       h->psd_grid_smem));
      if (occ < 1) throw Fail{SCS_ECUDA, "k_psd_grid: no resident CTA"};
      int per_sm = std::min(occ, 2);
      if (const char* e = getenv("SCS_PSD_GRID_PER_SM")) per_sm = std::max(1, std::min(occ, atoi(e)));
      // small sides: fewer CTAs (cheaper barriers), ~16 items per thread
      const long long items = (long long)kmax * kmax * 3 / 4;
      const long long want = (items + 16LL * kBlock - 1) / (16LL * kBlock);
      h->psd_grid_ctas = (int)std::max<long long>(1, std::min<long long>(want, (long long)h->sms * per_sm));
      h->psd_grid_part = dalloc<double>(h, h->psd_grid_ctas);
    }
  }
  {
    std::vector<int> cta;
    const int gmax = h->n_psd_grid > 0 ? h->psd_grid_max : 0;
    for (size_t b = 0; b < psd_side.size(); ++b) {
      const int k = psd_side[b];
      if (k <= h->warp_side || (k > h->smem_side && k <= gmax)) continue;
      cta.push_back((int)b);
    }
    h->n_psd_cta = (int)cta.size();
    if (!cta.empty()) h->psd_cta_list = up_i(cta);
    if (h->n_psd_cta + h->n_psd_small + h->n_psd_grid != (int)psd_side.size())
      throw Fail{SCS_EINVAL, "PSD block lists do not cover every block"};
  }
  if ((size_t)smem_optin(h, (const void*)k_cone_apply) < h->cone_smem)
    throw Fail{SCS_ECUDA, "k_cone_apply: shared memory budget exceeded"};
}

// ---------------------------------------------------------------------------
// matrices: CSC(A) is CSR(A^T) as-is; CSR(A) by a stable device radix sort
// ---------------------------------------------------------------------------
void build_matrices(scs_handle* h, const scs_problem* P) {
  const long long m = h->m, n = h->n, nnz = h->nnz;
  if (nnz >= (1LL << 31) - 1) throw Fail{SCS_EINVAL, "nnz >= 2^31 per shard is not supported"};
  if (m >= (1LL << 31) - 1 || n >= (1LL << 31) - 1)
    throw Fail{SCS_EINVAL, "dimensions >= 2^31 are not supported"};
  long long* tp = dalloc<long long>(h, n + 1);
  int* ti = dalloc<int>(h, nnz);
  double* tv = dalloc<double>(h, nnz);
  h2d(h, tp, (const long long*)P->colptr, n + 1);
  h2d(h, tv, P->vals, nnz);
  dbg("values copied (%.2f GB)", 8e-9 * (double)nnz);
  // row indices arrive as int64: stage in chunks and narrow on the device
  {
    const long long chunk = 1LL << 26;
    long long* stage = dalloc<long long>(h, std::min(chunk, std::max(nnz, 1LL)));
    for (long long o = 0; o < nnz; o += chunk) {
      const long long c = std::min(chunk, nnz - o);
      h2d(h, stage, (const long long*)P->rowidx + o, c);
      k_i64_to_i32<<<elem_grid(h, c), kBlock, 0, h->st>>>(stage, ti + o, c);
    }
    CK(cudaStreamSynchronize(h->st));
    dfree(h, stage);
  }
  dbg("row indices copied (%.2f GB)", 8e-9 * (double)nnz);
  h->At = Csr{tp, ti, tv, n};
  long long* rp = dalloc<long long>(h, m + 1);
  int* ci = dalloc<int>(h, nnz);
  double* av = dalloc<double>(h, nnz);
  if (nnz > 0) {
    int* colidx = dalloc<int>(h, nnz);
    k_expand_cols<<<elem_grid(h, n * 32), kBlock, 0, h->st>>>(tp, n, colidx);
    int* keys_out = dalloc<int>(h, nnz);
    int* perm_in = dalloc<int>(h, nnz);
    int* perm_out = dalloc<int>(h, nnz);
    k_iota<<<elem_grid(h, nnz), kBlock, 0, h->st>>>(perm_in, nnz);
    int bits = 1;
    while ((1LL << bits) < m) ++bits;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const int*)ti, keys_out,
                                       (const int*)perm_in, perm_out, (int)nnz, 0, bits, h->st));
    void* tmp = dalloc<char>(h, tmp_bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, (const int*)ti, keys_out,
                                       (const int*)perm_in, perm_out, (int)nnz, 0, bits, h->st));
    k_rowptr<<<elem_grid(h, m + 1), kBlock, 0, h->st>>>(keys_out, nnz, m, rp);
    k_gather_csr<<<elem_grid(h, nnz), kBlock, 0, h->st>>>(perm_out, colidx, tv, nnz, ci, av);
    CK(cudaStreamSynchronize(h->st));
    dfree(h, tmp);
    dfree(h, perm_out);
    dfree(h, perm_in);
    dfree(h, keys_out);
    dfree(h, colidx);
  } else {
    CK(cudaMemsetAsync(rp, 0, (m + 1) * sizeof(long long), h->st));
  }
  h->A = Csr{rp, ci, av, m};
  h->LA = pick_lanes(nnz, m);
  h->LAt = pick_lanes(nnz, n);
  if (const char* e = getenv("SCS_LANES_A")) h->LA = atoi(e);     // tuning overrides
  if (const char* e = getenv("SCS_LANES_AT")) h->LAt = atoi(e);
}

double dev_scalar(scs_handle* h, int idx = 0) {
  double v = 0.0;
  CK(cudaMemcpyAsync(&v, h->dscal + idx, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return v;
}

// sum over a vector (mode 0: (a b)^2, 1: (a/b)^2, 2: a b); `ysum` = the
// vector is row-sharded, so the shard totals are all-reduced
double norm2_dev(scs_handle* h, const double* a, const double* b, long long n, int mode,
                 bool ysum = false) {
  k_norm2<<<elem_grid(h, n), kBlock, 0, h->st>>>(a, b, n, mode, h->V.part, &h->ctl->counter,
                                                   h->dscal);
  if (ysum) allreduce(h, h->dscal, 1);
  return dev_scalar(h);
}

// ---------------------------------------------------------------------------
// equilibration (scaling.py:79-129) -- D, E from A only; sigma, rho need b, c
// ---------------------------------------------------------------------------
void equilibrate(scs_handle* h) {
  const long long m = h->m, n = h->n, nnz = h->nnz;
  double* cn = h->tmp_n;
  double* rn = h->tmp_m;
  double* cs = h->V.Gp;  // scratch n
  double* rs = h->tmp_m2;
  {
    std::vector<double> ones(std::max(m, n), 1.0);
    h2d(h, h->D, ones.data(), m);
    h2d(h, h->E, ones.data(), n);
    CK(cudaStreamSynchronize(h->st));
  }
  const long long zl = h->K.z + h->K.l;
  auto col_norms = [&]() {  // sqrt of all-reduced column sums of squares
    k_row_sumsq<<<elem_grid(h, n * 32), kBlock, 0, h->st>>>(h->At, cn);
    allreduce(h, cn, n);
  };
  auto row_norms = [&]() {
    k_row_sumsq<<<elem_grid(h, m * 32), kBlock, 0, h->st>>>(h->A, rn);
    k_sqrt<<<elem_grid(h, m), kBlock, 0, h->st>>>(rn, m);
  };
  auto seg_means = [&]() {
    CK(cudaMemsetAsync(h->seg_sum, 0, std::max(h->nseg_g, 1) * sizeof(double), h->st));
    k_seg_partial<<<std::max(1, std::min(h->nseg, h->grid_full)), kBlock, 0, h->st>>>(
        rn, h->nseg, h->seg_off, h->seg_len, h->seg_gid, h->seg_sum);
    allreduce(h, h->seg_sum, h->nseg_g);
    k_seg_means<<<elem_grid(h, h->nseg_g), kBlock, 0, h->st>>>(h->seg_sum, h->seg_glen, h->nseg_g,
                                                                 h->seg_mean);
  };
  if (h->set.normalize) {
    for (int sw = 0; sw < h->set.sweeps; ++sw) {
      col_norms();
      k_inv_sqrt_scale<<<elem_grid(h, n), kBlock, 0, h->st>>>(cn, n, cs, h->E);
      k_scale_rows<<<elem_grid(h, n * 32), kBlock, 0, h->st>>>((long long*)h->At.rp,
                                                                (double*)h->At.v, n, cs);
      k_scale_cols<<<elem_grid(h, nnz), kBlock, 0, h->st>>>(h->A.ci, (double*)h->A.v, nnz, cs);
      row_norms();
      seg_means();
      k_block_rows<<<elem_grid(h, std::max<long long>(zl, (long long)h->nseg * kBlock)), kBlock, 0,
                     h->st>>>(rn, zl, h->nseg, h->seg_off, h->seg_len, h->seg_gid, h->seg_mean,
                              rs, h->D);
      k_scale_rows<<<elem_grid(h, m * 32), kBlock, 0, h->st>>>((long long*)h->A.rp,
                                                                (double*)h->A.v, m, rs);
      k_scale_cols<<<elem_grid(h, nnz), kBlock, 0, h->st>>>(h->At.ci, (double*)h->At.v, nnz, rs);
    }
    col_norms();
    k_sqrt<<<elem_grid(h, n), kBlock, 0, h->st>>>(cn, n);  // replicated on every shard
    k_pos_mean<<<elem_grid(h, n), kBlock, 0, h->st>>>(cn, n, h->V.part, &h->ctl->counter, h->dscal);
    double s0 = dev_scalar(h, 0), c0 = dev_scalar(h, 1);
    h->mean_col = c0 > 0 ? s0 / c0 : 1.0;
    row_norms();
    seg_means();
    k_pos_mean<<<elem_grid(h, zl), kBlock, 0, h->st>>>(rn, zl, h->V.part, &h->ctl->counter, h->dscal);
    allreduce(h, h->dscal, 2);
    double s1 = dev_scalar(h, 0), c1 = dev_scalar(h, 1);
    k_pos_mean<<<elem_grid(h, h->nseg_g), kBlock, 0, h->st>>>(h->seg_mean, h->nseg_g, h->V.part,
                                                               &h->ctl->counter, h->dscal);
    double s2 = dev_scalar(h, 0), c2 = dev_scalar(h, 1);
    h->mean_row = (c1 + c2) > 0 ? (s1 + s2) / (c1 + c2) : 1.0;
  } else {
    h->mean_col = h->mean_row = 1.0;
  }
  CK(cudaStreamSynchronize(h->st));
}

void pull_ctl(scs_handle* h) {
  CK(cudaMemcpyAsync(h->ctl_h, h->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
}
void push_ctl(scs_handle* h) {
  CK(cudaMemcpyAsync(h->ctl, h->ctl_h, sizeof(Ctl), cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
}

// sigma, rho, b_hat, c_hat and the residual constants (scaling.py:121-128,
// 469-478)
void scale_vectors(scs_handle* h) {
  const long long m = h->m, n = h->n;
  if (h->set.normalize) {
    const double dbn = sqrt(norm2_dev(h, h->D, h->b0, m, 0, true));
    const double ecn = sqrt(norm2_dev(h, h->E, h->c0, n, 0));
    h->sigma = dbn > 0 ? h->mean_col / dbn : 1.0;
    h->rho = ecn > 0 ? h->mean_row / ecn : 1.0;
  } else {
    h->sigma = h->rho = 1.0;
  }
  k_scale_vec<<<elem_grid(h, m), kBlock, 0, h->st>>>(h->b0, h->D, h->sigma, m, h->bh);
  k_scale_vec<<<elem_grid(h, n), kBlock, 0, h->st>>>(h->c0, h->E, h->rho, n, h->ch);
  const double dib = sqrt(norm2_dev(h, h->bh, h->D, m, 1, true));
  const double eic = sqrt(norm2_dev(h, h->ch, h->E, n, 1));
  pull_ctl(h);
  Ctl* c = h->ctl_h;
  c->b_norm = dib / h->sigma;
  c->c_norm = eic / h->rho;
  c->b_ref = dib > 0 ? dib : 1.0;
  c->c_ref = eic > 0 ? eic : 1.0;
  c->sigma = h->sigma;
  c->rho = h->rho;
  push_ctl(h);
}

void check_err(scs_handle* h) {
  const int e = h->ctl_h->err;
  if (!e) return;
  if (e & ERR_CG_CURVATURE)
    throw Fail{SCS_ENONFINITE, "cg_solve: operator is not positive definite on iterates"};
  if (e & ERR_CG_NONFINITE) throw Fail{SCS_ENONFINITE, "cg_solve: non-finite residual"};
  if (e & ERR_CONE_NONFINITE) throw Fail{SCS_ENONFINITE, "project_embedding_cone: non-finite input"};
  if (e & ERR_SCHED)
    throw Fail{SCS_ECUDA, "internal: iteration graph variant does not match the refresh schedule"};
  if (e & ERR_JACOBI) {
    if (h->V.dbg) {
      const int cap = 2 + h->K.max_side * (h->K.max_side + 1) / 2;
      std::vector<double> d(cap);
      cudaMemcpy(d.data(), h->V.dbg, cap * sizeof(double), cudaMemcpyDeviceToHost);
      const int k = (int)d[1];
      fprintf(stderr, "[scs] non-converged PSD block side %d svec:", k);
      for (int i = 0; i < k * (k + 1) / 2; ++i) fprintf(stderr, " %.17g", d[2 + i]);
      fprintf(stderr, "\n");
    }
    throw Fail{SCS_ENOCONV, "Jacobi eigensolver did not converge within 100 sweeps"};
  }
}

// one CG step (A p, A^T, update, p update); the first step of an ADMM
// iteration also closes the previous iteration's termination check
void cg_step(scs_handle* h, const Vec& V, long long cap, bool with_p, bool merged, bool recur) {
  // residual recurrence (V.Agx set): the merged pass runs on refresh
  // iterations only (and stores A u_x); the others check from Aux and run
  // a plain A p pass
  const int R = (merged && V.Agx) ? h->res_rec : 0;
  if (merged && !h->stm_m[0]) {  // CSR: plain SpMV + elementwise residual pass
    EpiApPlain2 ea{};
    ea.V = V;
    ea.xb = V.X2;
    ea.rgate = R;
    ea.waux = R > 0;
    launch_mat(h, 0, ea);
    EpiResY ry{};
    ry.V = V;
    ry.rgate = R;
    y_rows(h, V.Aux, ry);
  } else if (merged) {
    EpiAp<true> ea{};
    ea.V = V;
    ea.xb = V.X2;
    ea.rgate = R;
    ea.waux = R > 0;
    a_pass(h, ea);
  }
  if (merged && R > 0) {
    EpiResY ry{};
    ry.V = V;
    ry.rgate = -R;
    y_rows(h, V.Aux, ry);
    EpiAp<false> ea{};
    ea.V = V;
    ea.xb = V.P1;
    ea.rgate = -R;
    a_pass(h, ea);
  } else if (!merged) {
    EpiAp<false> ea{};
    ea.V = V;
    ea.xb = V.P1;
    a_pass(h, ea);
  }
  EpiAtGp eg{};
  eg.V = V;
  eg.xb = V.q;
  at_pass(h, eg);
  k_cg_update<<<elem_grid(h, recur ? std::max(h->n, h->m) : h->n), kBlock, 0, h->st>>>(V, cap,
                                                                                    recur ? 1 : 0);
  h->launches++;
  if (with_p) {
    k_cg_p<<<elem_grid(h, h->n), kBlock, 0, h->st>>>(V);
    h->launches++;
  }
}

// g = M^-1 h by CG to 1e-9 (1 + ||h||) from zero (embedding.py:145-162)
void solve_g(scs_handle* h) {
  const long long n = h->n, m = h->m;
  Vec G = h->V;
  G.T = nullptr;  // the g solve's CG must not touch the iteration's A^T A x
  G.rhs_x = h->ch;
  G.x = h->V.gx;
  G.rhs_y = h->bh;
  k_zero<<<elem_grid(h, n), kBlock, 0, h->st>>>(G.x, n);
  k_fill_y2<<<elem_grid(h, m), kBlock, 0, h->st>>>(G.Y2, h->bh, m);
  const double hn = sqrt(norm2_dev(h, h->ch, h->ch, n, 2) + norm2_dev(h, h->bh, h->bh, m, 2, true));
  pull_ctl(h);
  Ctl* c = h->ctl_h;
  c->stop = 0;
  c->err = 0;
  c->tol = 1e-9 * (1.0 + hn);
  c->cg_done = 0;
  c->cg_it = 0;
  c->counter = 0;
  c->check_pending = 0;
  c->force_check = 0;
  push_ctl(h);
  const long long cap = 10 * n + 100;  // embedding.py:104
  EpiAtFirst e0{};
  e0.V = G;
  e0.xb = G.Y2;
  at_pass(h, e0);
  long long done_steps = 0;
  while (true) {
    pull_ctl(h);
    dbg("g-solve: steps=%lld cg_it=%d done=%d err=%d", done_steps, c->cg_it, c->cg_done, c->err);
    check_err(h);
    if (c->cg_done) break;
    const long long batch = std::min<long long>(32, cap - done_steps);
    if (batch <= 0) break;
    for (long long i = 0; i < batch; ++i) cg_step(h, G, cap, true, false, false);
    done_steps += batch;
  }
  a_final(h, G, h->V.gy, 1);
  if (h->V.Agx) {  // A g_x for the residual recurrence
    EpiPlain e{};
    e.V = h->V;
    e.xb = h->V.gx;
    e.out = h->V.Agx;
    launch_mat(h, 0, e);
  }
  if (h->V.T) {  // A^T b^ and A^T g_y for the A^T-side recurrence
    EpiPlain e{};
    e.V = h->V;
    e.xb = h->bh;
    e.out = h->V.Atb;
    at_pass(h, e);
    e.xb = h->V.gy;
    e.out = h->V.Atgy;
    at_pass(h, e);
  }
  pull_ctl(h);
  check_err(h);
  if (c->denom < 1.0 - 1e-9)
    throw Fail{SCS_ESETUP, "Schur denominator " + std::to_string(c->denom) + " below 1"};
}

void launch_cone_apply(scs_handle* h, const Vec& V);

// one ADMM iteration: the kernel sequence of kernels.cuh (with all-reduces
// between kernels when rows are sharded)
void enqueue_iteration(scs_handle* h) {
  const Vec V = h->V;
  k_prep<<<elem_grid(h, h->n + h->m), kBlock, 0, h->st>>>(V, h->sharded ? 1 : 0, h->variant,
                                                          std::max(h->R, 1));
  h->launches++;
  if (h->sharded) {
    allreduce(h, V.dred, 1);
    k_prep_finish<<<1, 32, 0, h->st>>>(V, h->variant, std::max(h->R, 1));
    h->launches++;
  }
  const int RA = V.T ? h->res_rec : 0;  // A^T-side residual recurrence
  if (RA) {
    EpiTRef et{};
    et.V = V;
    et.xb = V.Axw;
    et.rgate = RA;
    at_pass(h, et);
  }
  EpiAtFirst e0{};
  e0.V = V;
  e0.xb = V.Y2;
  e0.rgate = RA;
  at_pass(h, e0);
  if (RA && !gated_off(h, -RA)) {
    EpiAtFirst1 e1{};
    e1.V = V;
    e1.xb = V.Yc;
    e1.rgate = -RA;
    if (!h->sharded) {  // products into Sv, then the epilogue coalesced
      EpiStoreF sf{};
      sf.V = V;
      sf.xb = V.Yc;
      sf.rgate = -RA;
      int sp = 1;
      if (h->stm_m[1] && ((uintptr_t)sf.xb & 15) == 0)  // split partials summed by k_rows below
        sp = launch_stream<1, 1, EpiStoreF>(h, 1, sf, -1, false);
      else
        launch_mat(h, 1, sf);
      k_rows<EpiAtFirst1><<<elem_grid(h, h->n), kBlock, 0, h->st>>>(sp > 1 ? h->Pstm : V.Sv, h->n, sp,
                                                                     e1);
      h->launches++;
    } else {
      at_pass(h, e1);
    }
  }
  const long long cgm = h->set.cg_max;
  const bool recur = (h->set.fast & SCS_FAST_RECURRENCE) != 0;
  for (long long i = 0; i < cgm; ++i) cg_step(h, V, cgm, i + 1 < cgm, i == 0, recur);
  a_final(h, V, V.zy, 0);
  const long long work = std::max<long long>(h->n + h->K.z + h->K.l, 1);
  int g_tail = std::max(elem_grid(h, work), std::min(h->K.n_chunk, h->grid_full));
  g_tail = std::max(g_tail, std::min((int)((h->K.n_ssoc * 32LL + kBlock - 1) / kBlock), h->grid_full));
  k_cone_tail<<<g_tail, kBlock, 0, h->st>>>(V, h->K, h->sharded ? 1 : 0);
  h->launches++;
  if (h->sharded) {
    allreduce(h, V.cone_red, h->cone_red_len);
    k_cone_finish<<<1, kBlock, 0, h->st>>>(V, h->K);
    h->launches++;
  }
  launch_cone_apply(h, V);
}

// big SOCs and large PSD blocks (CTA each), then small PSD blocks (warp each)
void launch_cone_apply(scs_handle* h, const Vec& V) {
  const int n_big = h->n_psd_cta;
  if (h->K.n_chunk > 0 || n_big > 0) {
    const int g = std::max(1, std::min(std::max(h->K.n_chunk, n_big), h->grid_full));
    k_cone_apply<<<g, kBlock, h->cone_smem, h->st>>>(V, h->K, h->psd_scratch, h->smem_side,
                                                      h->psd_cta_list, h->n_psd_cta);
    h->launches++;
  }
  if (h->n_psd_small > 0) {
    const long long g = std::min<long long>((h->n_psd_small + kBlock / 32 - 1) / (kBlock / 32),
                                            (long long)h->sms * 32);
    k_psd_small<<<(int)g, kBlock, kPsdSmallSmem, h->st>>>(V, h->K, h->psd_small_list,
                                                          h->n_psd_small);
    h->launches++;
  }
  if (h->n_psd_grid > 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->psd_grid_ctas);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = h->psd_grid_smem;
    cfg.stream = h->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_psd_grid, V, h->K, h->psd_scratch, h->psd_grid_list,
                          h->n_psd_grid, h->psd_grid_part));
    h->launches++;
  }
}

// Capture one ADMM iteration of the given variant into a CUDA graph (NCCL
// calls are capturable; the emulated group is not, and runs the sequence
// directly).
cudaGraphExec_t capture_iteration(scs_handle* h, int variant, long long* lpi) {
  const long long before = h->launches;
  h->variant = variant;
  CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  enqueue_iteration(h);
  cudaGraph_t g;
  CK(cudaStreamEndCapture(h->st, &g));
  h->variant = 0;
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  *lpi = h->launches - before;
  h->launches = before;
  return ex;
}

__global__ void k_loop_arm(Ctl* c, cudaGraphConditionalHandle wh) {
  c->loop_done = 0;
  c->loop_refresh = 0;
  cudaGraphSetConditional(wh, (c->loop_left > 0 && !c->stop) ? 1u : 0u);
}

// One GPU: the whole loop as one graph --
//   [k_loop_arm] -> WHILE { [k_loop_pick] -> SWITCH { non-refresh iteration,
//                                                     refresh iteration }
//                           -> [k_loop_next] }
// (no SWITCH when the residual recurrences are off).  The host writes the
// iteration budget into Ctl.loop_left (8-byte copy) before each launch.
// Returns false (and leaves gloop unset) if the driver rejects the graph.
bool build_loop_graph(scs_handle* h) {
  const cudaStreamCaptureMode mode = cudaStreamCaptureModeThreadLocal;
  cudaGraph_t g = nullptr;
  CK(cudaGraphCreate(&g, 0));
  auto fail = [&](const char* what, cudaError_t e) {
    dbg("loop graph: %s failed: %s", what, cudaGetErrorString(e));
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(h->st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(h->st, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGetLastError();
    h->variant = 0;
    cudaGraphDestroy(g);
    return false;
  };
  cudaError_t e;
  cudaGraphConditionalHandle wh;
  if ((e = cudaGraphConditionalHandleCreate(&wh, g, 0, 0)) != cudaSuccess) return fail("handle", e);
  if ((e = cudaStreamBeginCaptureToGraph(h->st, g, nullptr, nullptr, 0, mode)) != cudaSuccess)
    return fail("capture arm", e);
  k_loop_arm<<<1, 1, 0, h->st>>>(h->ctl, wh);
  if ((e = cudaStreamEndCapture(h->st, &g)) != cudaSuccess) return fail("end arm", e);
  cudaGraphNode_t arm = nullptr;
  size_t nn = 1;
  if ((e = cudaGraphGetNodes(g, &arm, &nn)) != cudaSuccess || nn != 1) return fail("arm node", e);
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = wh;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  if ((e = cudaGraphAddNode(&wnode, g, &arm, 1, &wp)) != cudaSuccess) return fail("while", e);
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphNode_t last = nullptr;
  const long long before = h->launches;
  if (h->R > 0) {
    cudaGraphConditionalHandle sh;
    if ((e = cudaGraphConditionalHandleCreate(&sh, body, 0, 0)) != cudaSuccess)
      return fail("switch handle", e);
    if ((e = cudaStreamBeginCaptureToGraph(h->st, body, nullptr, nullptr, 0, mode)) != cudaSuccess)
      return fail("capture pick", e);
    k_loop_pick<<<1, 1, 0, h->st>>>(h->ctl, sh, h->R);
    if ((e = cudaStreamEndCapture(h->st, &body)) != cudaSuccess) return fail("end pick", e);
    cudaGraphNode_t pick = nullptr;
    nn = 1;
    if ((e = cudaGraphGetNodes(body, &pick, &nn)) != cudaSuccess || nn != 1)
      return fail("pick node", e);
    cudaGraphNodeParams sp{};
    sp.type = cudaGraphNodeTypeConditional;
    sp.conditional.handle = sh;
    sp.conditional.type = cudaGraphCondTypeSwitch;
    sp.conditional.size = 2;
    if ((e = cudaGraphAddNode(&last, body, &pick, 1, &sp)) != cudaSuccess) return fail("switch", e);
    for (int b = 0; b < 2; ++b) {
      cudaGraph_t br = sp.conditional.phGraph_out[b];
      if ((e = cudaStreamBeginCaptureToGraph(h->st, br, nullptr, nullptr, 0, mode)) != cudaSuccess)
        return fail("capture branch", e);
      h->variant = b ? 2 : 1;
      enqueue_iteration(h);
      h->variant = 0;
      if ((e = cudaStreamEndCapture(h->st, &br)) != cudaSuccess) return fail("end branch", e);
    }
    if ((e = cudaStreamBeginCaptureToGraph(h->st, body, &last, nullptr, 1, mode)) != cudaSuccess)
      return fail("capture next", e);
  } else {
    if ((e = cudaStreamBeginCaptureToGraph(h->st, body, nullptr, nullptr, 0, mode)) != cudaSuccess)
      return fail("capture body", e);
    enqueue_iteration(h);
  }
  k_loop_next<<<1, 1, 0, h->st>>>(h->ctl, wh);
  if ((e = cudaStreamEndCapture(h->st, &body)) != cudaSuccess) return fail("end body", e);
  h->launches = before;
  cudaGraphExec_t ex = nullptr;
  if ((e = cudaGraphInstantiate(&ex, g, 0)) != cudaSuccess) return fail("instantiate", e);
  cudaGraphDestroy(g);
  h->gloop = ex;
  return true;
}

void destroy_graphs(scs_handle* h) {
  for (auto* ex : {&h->gvar[0], &h->gvar[1], &h->gloop})
    if (*ex) { cudaGraphExecDestroy(*ex); *ex = nullptr; }
}

// The iteration graphs: with the residual recurrences on, one graph per
// variant (refresh iterations k_sched = 1, 1 + R, ... carry the direct
// residual passes, the others the recurrence passes), so no gated-off pass
// is launched (and, row-sharded, no all-reduce of a gated-off pass runs).
// On one GPU, also the device-side loop over them (build_loop_graph).
void build_graph(scs_handle* h) {
  destroy_graphs(h);
  h->R = (h->V.Agx || h->V.T) ? h->res_rec : 0;
  if (!h->use_graph) {
    h->launches_per_iter = 0;
    return;
  }
  if (h->R > 0) {
    h->gvar[0] = capture_iteration(h, 1, &h->lpi_var[0]);
    h->gvar[1] = capture_iteration(h, 2, &h->lpi_var[1]);
  } else {
    h->gvar[0] = capture_iteration(h, 0, &h->lpi_var[0]);
    h->lpi_var[1] = h->lpi_var[0];
  }
  h->launches_per_iter = h->lpi_var[0];
  if (!h->sharded && env_ll("SCS_LOOP_GRAPH", 1)) build_loop_graph(h);
  dbg("graphs: R=%d launches/iter %lld (refresh %lld), loop graph %d", h->R, h->lpi_var[0],
      h->lpi_var[1], h->gloop != nullptr);
}

// One iteration from the host: the variant follows the refresh schedule,
// predicted from the iterations launched since scs_begin (k_sched before
// this iteration; k_prep verifies the prediction on the device).
void run_iteration(scs_handle* h) {
  const int refresh = (h->R > 0 && h->launched_iters % h->R == 0) ? 1 : 0;
  if (h->use_graph) {
    CK(cudaGraphLaunch(h->gvar[h->R > 0 ? refresh : 0], h->st));
    h->launches += h->lpi_var[refresh];
  } else {
    const long long before = h->launches;
    h->variant = h->R > 0 ? 1 + refresh : 0;
    enqueue_iteration(h);
    h->variant = 0;
    h->launches_per_iter = h->launches - before;
  }
  h->launched_iters++;
}

// Up to k iterations as one launch of the loop graph (stops on the device
// at termination or error); returns after the graph is enqueued.
void enqueue_loop(scs_handle* h, long long k) {
  *h->loop_arg = k;
  CK(cudaMemcpyAsync(&h->ctl->loop_left, h->loop_arg, sizeof(long long), cudaMemcpyHostToDevice,
                     h->st));
  CK(cudaGraphLaunch(h->gloop, h->st));
}

// bookkeeping after a loop launch (Ctl pulled)
void account_loop(scs_handle* h) {
  const Ctl* c = h->ctl_h;
  const long long done = c->loop_done, refr = c->loop_refresh;
  h->launched_iters += done;
  // the iterations' kernels, k_loop_next (+ k_loop_pick) per iteration, k_loop_arm
  h->launches += (done - refr) * h->lpi_var[0] + refr * h->lpi_var[1] + done +
                 (h->R > 0 ? done : 0) + 1;
}

// stand-alone termination check / residual evaluation of the current state
// (the products are kept: A u_x in V.Aux, A^T u_y in V.Uy when allocated)
void launch_residuals(scs_handle* h) {
  EpiResA ra{};
  ra.V = h->V;
  ra.xb = h->V.u;
  ra.store = h->V.Aux;
  a_pass(h, ra);
  EpiResAt rt{};
  rt.V = h->V;
  rt.xb = h->V.u + h->n;
  rt.store = h->V.Uy;
  at_pass(h, rt);
}

void fill_info(scs_handle* h, scs_info* info) {
  if (!info) return;
  const Ctl* c = h->ctl_h;
  info->status = c->status;
  info->iterations = c->iter;
  info->cg_iters = c->cg_iters_total;
  for (int i = 0; i < 8; ++i) info->res[i] = c->res[i];
  info->setup_seconds = h->setup_seconds;
  info->launches = h->launches;
}

void do_begin(scs_handle* h, const double* wx, const double* wy, const double* ws) {
  const long long n = h->n, m = h->m;
  h->prod_current = false;
  double *dx = nullptr, *dy = nullptr, *ds = nullptr;
  if (wx) {
    dx = h->tmp_n;
    dy = h->tmp_m;
    ds = h->tmp_m2;
    h2d(h, dx, wx, n);
    h2d(h, dy, wy, m);
    h2d(h, ds, ws, m);
  }
  k_init_state<<<elem_grid(h, n + m + 1), kBlock, 0, h->st>>>(h->V, dx, dy, ds, h->sigma, h->rho);
  pull_ctl(h);
  Ctl* c = h->ctl_h;
  c->iter = 0;
  c->k_sched = 0;  // reset_schedule (embedding.py:45-48)
  c->status = SCS_RUNNING;
  c->stop = 0;
  c->err = 0;
  c->warm_zero = 1;
  c->force_check = 0;
  c->check_pending = 0;
  c->counter = 0;
  c->max_iters = h->set.max_iters;
  c->check_interval = h->set.check_interval;
  push_ctl(h);
  h->launched_iters = 0;
  h->launches = 0;
}

// Row-sharded: a Jacobi non-convergence is detected on the rank that owns
// the PSD block only; OR the error bits over all ranks at every batch end so
// that every rank raises after the same batch (instead of the others
// waiting in the next collective).
__global__ void k_err_pack(Ctl* c, double* d) {
  if (threadIdx.x < 4) d[threadIdx.x] = (c->err >> threadIdx.x) & 1 ? 1.0 : 0.0;
}
__global__ void k_err_unpack(Ctl* c, const double* d) {
  if (threadIdx.x) return;
  int e = 0;
  for (int b = 0; b < 4; ++b) e |= d[b] > 0.0 ? 1 << b : 0;
  if (e) { c->err |= e; c->stop = 1; }
}
void share_err(scs_handle* h) {
  if (!h->sharded) return;
  k_err_pack<<<1, 32, 0, h->st>>>(h->ctl, h->dscal);
  allreduce(h, h->dscal, 4);
  k_err_unpack<<<1, 32, 0, h->st>>>(h->ctl, h->dscal);
}

// run up to k iterations, stopping at termination or max_iters
void do_steps(scs_handle* h, long long k) {
  Ctl* c = h->ctl_h;
  long long todo = std::min(k, h->set.max_iters - h->launched_iters);
  if (todo > 0 && h->gloop) {  // one launch, the loop runs on the device
    enqueue_loop(h, todo);
    pull_ctl(h);
    account_loop(h);
    dbg("loop: launched=%lld iter=%lld status=%d stop=%d err=%d", h->launched_iters, c->iter,
        c->status, c->stop, c->err);
    check_err(h);
    return;
  }
  long long batch = 1;
  while (todo > 0) {
    const long long b = std::min(batch, todo);
    for (long long i = 0; i < b; ++i) run_iteration(h);
    todo -= b;
    share_err(h);
    pull_ctl(h);
    dbg("steps: launched=%lld iter=%lld status=%d stop=%d err=%d cg_it=%d", h->launched_iters,
        c->iter, c->status, c->stop, c->err, c->cg_it);
    check_err(h);
    if (c->stop) break;
    batch = std::min<long long>(batch * 2, 64);
  }
}

// Loop exit (solver.py:359-369): the last iteration's termination check is
// still pending (it normally rides on the next iteration's first passes);
// run it stand-alone, then apply the post-loop status rule.
void do_finish(scs_handle* h) {
  Ctl* c = h->ctl_h;
  pull_ctl(h);
  // V.Aux / V.Uy end up holding A_hat u_x / A_hat^T u_y of the final state:
  // from the check that stopped the loop (direct on refresh iterations, else
  // by the recurrences), or from launch_residuals below
  h->prod_current = h->R > 0 && h->V.Uy != nullptr;
  if (c->status != SCS_RUNNING) return;
  bool fresh = false;
  if (c->check_pending && !c->stop) {
    launch_residuals(h);
    pull_ctl(h);
    check_err(h);
    if (c->status != SCS_RUNNING) return;
    fresh = true;  // Ctl.res already holds the final state's residuals
  }
  if (!fresh) {  // post-loop residuals (solver.py:365) of a state that was not checked
    c->force_check = 1;
    c->stop = 0;
    push_ctl(h);
    launch_residuals(h);
  }
  // tau > 1e-8 ||u|| ?  (x-part and tau replicated, y-part sharded)
  const long long n = h->n, m = h->m;
  const double un2 = norm2_dev(h, h->V.u, h->V.u, n, 2) +
                     norm2_dev(h, h->V.u + n, h->V.u + n, m, 2, true);
  pull_ctl(h);
  double ut = 0.0;
  d2h(h, &ut, h->V.u + n + m, 1);
  CK(cudaStreamSynchronize(h->st));
  const double un = sqrt(un2 + ut * ut);
  c->status = ut > 1e-8 * un ? SCS_MAX_ITERS_REACHED : SCS_INDETERMINATE;
  c->force_check = 0;
  c->stop = 1;
  push_ctl(h);
}

int guard(scs_handle* h, const std::function<void()>& fn) {
  try {
    if (h) CK(cudaSetDevice(h->dev));
    fn();
    return SCS_OK;
  } catch (const Fail& f) {
    if (h) h->err = f.msg;
    set_global_err(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    if (h) h->err = e.what();
    set_global_err(e.what());
    return SCS_ENOMEM;
  }
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int scs_abi_version(void) { return SCS_B200_ABI_VERSION; }

const char* scs_last_error(const scs_handle* h) {
  if (h) return h->err.c_str();
  std::lock_guard<std::mutex> g(g_err_mu);
  return g_err.c_str();
}

void scs_destroy(scs_handle* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  destroy_graphs(h);
  for (auto& b : h->bufs)
    if (b.p) {
      if (h->st) cudaFreeAsync(b.p, h->st);
      else cudaFree(b.p);
    }
  if (h->st) cudaStreamSynchronize(h->st);
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, h->dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    cudaGetLastError();
  }
  if (h->ctl_h) cudaFreeHost(h->ctl_h);
  free_stage(h);
  if (h->loop_arg) cudaFreeHost(h->loop_arg);
  if (h->st) cudaStreamDestroy(h->st);
  if (h->st_copy) cudaStreamDestroy(h->st_copy);
  if (h->st_comm) cudaStreamDestroy(h->st_comm);
  for (auto& e : h->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (h->ev_comm) cudaEventDestroy(h->ev_comm);
  delete h->comm;
  delete h;
}

scs_emu_group* scs_emu_group_create(int32_t world) {
  if (world < 1) return nullptr;
  scs_emu_group* g = new scs_emu_group();
  g->world = world;
  g->ptr.assign(world, nullptr);
  g->cnt.assign(world, 0);
  return g;
}

void scs_emu_group_destroy(scs_emu_group* g) { delete g; }

static void validate(const scs_problem* P, const scs_settings* S) {
  if (!P || !S) throw Fail{SCS_EINVAL, "null problem or settings"};
  if (P->m < 0 || P->n < 0) throw Fail{SCS_EINVAL, "matrix dimensions must be nonnegative"};
  if (!(S->alpha > 0.0 && S->alpha < 2.0)) throw Fail{SCS_EINVAL, "alpha must lie in (0, 2)"};
  const double eps[5] = {S->eps_pri, S->eps_dual, S->eps_gap, S->eps_infeas, S->eps_unbdd};
  for (double e : eps)
    if (!(e > 0)) throw Fail{SCS_EINVAL, "eps must be positive"};
  if (S->max_iters < 1 || S->check_interval < 1)
    throw Fail{SCS_EINVAL, "max_iters and check_interval must be >= 1"};
  if (S->cg_max < 1) throw Fail{SCS_EINVAL, "cg_max must be >= 1"};
  if (S->sweeps < 0) throw Fail{SCS_EINVAL, "sweeps must be >= 0"};
  if (S->fast & ~(SCS_FAST_PCG | SCS_FAST_RECURRENCE)) throw Fail{SCS_EINVAL, "unknown fast-mode bits"};
  if (P->z < 0 || P->l < 0 || P->ep < 0) throw Fail{SCS_EINVAL, "cone dimensions must be nonnegative"};
  if (P->colptr[0] != 0) throw Fail{SCS_EINVAL, "colptr must start at 0 and end at nnz"};
  for (long long j = 0; j < P->n; ++j)
    if (P->colptr[j + 1] < P->colptr[j]) throw Fail{SCS_EINVAL, "colptr must be nondecreasing"};
}

int scs_create(const scs_problem* P, const scs_settings* S, const scs_dist* dist,
               scs_handle** out) {
  if (!out) return SCS_EINVAL;
  *out = nullptr;
  scs_handle* h = new scs_handle();
  Timer tm;
  int rc = guard(nullptr, [&] {
    dbg("scs_create enter");
    validate(P, S);
    dbg("validated");
    h->set = *S;
    if (const char* e = getenv("SCS_RECUR_REFRESH")) h->recur_refresh = std::max(1, atoi(e));
    if (const char* e = getenv("SCS_RES_RECUR")) h->res_rec = std::max(0, atoi(e));
    if (const char* e = getenv("SCS_RES_RECUR_AT")) h->res_rec_at = atoi(e) != 0;
    h->dev = S->device;
    CK(cudaSetDevice(h->dev));
    CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->dev));
    h->grid_full = h->sms * (2048 / kBlock);
    if (h->grid_full > kMaxGrid) h->grid_full = kMaxGrid;
    CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->st_copy, cudaStreamNonBlocking));
    {
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, h->dev));
      unsigned long long keep = ~0ull;  // freed blocks stay in the pool (trimmed at destroy)
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    {
      // opt-in (SCS_L2_PERSIST=1): measured slower at config 5 -- the
      // set-aside shrinks the L2 left for everything else
      const char* env = getenv("SCS_L2_PERSIST");
      int maxp = 0, maxw = 0;
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, h->dev);
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, h->dev);
      if (env && atoi(env) != 0 && maxp > 0 && maxw > 0 &&
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) == cudaSuccess) {
        h->l2_persist = (size_t)maxp;
        h->l2_window_max = (size_t)maxw;
      }
      cudaGetLastError();
      dbg("L2 persisting set-aside %zu bytes, window max %zu", h->l2_persist, h->l2_window_max);
    }
    h->m = P->m;
    h->n = P->n;
    h->m_glob = P->m_global > 0 ? P->m_global : P->m;
    h->row_lo = P->row_lo;
    h->nnz = P->colptr[P->n];
    const long long m = h->m, n = h->n;
    h->bounds = {0, h->m_glob};
    if (dist) {
      h->rank = dist->rank;
      h->world = dist->world;
      if (h->world < 1 || h->rank < 0 || h->rank >= h->world)
        throw Fail{SCS_EINVAL, "bad rank/world"};
      if (dist->bounds) h->bounds.assign(dist->bounds, dist->bounds + h->world + 1);
      else if (h->world > 1) throw Fail{SCS_EINVAL, "row-sharded create needs the shard bounds"};
      if (h->bounds[h->rank] != h->row_lo || h->bounds[h->rank + 1] - h->bounds[h->rank] != m ||
          h->bounds.front() != 0 || h->bounds.back() != h->m_glob)
        throw Fail{SCS_EINVAL, "shard bounds do not match row_lo / m / m_global"};
      h->sharded = h->world > 1 || (dist->flags & SCS_DIST_FORCE);
      if (h->sharded) {
        if (dist->emu_group) {
          scs_emu_group* g = (scs_emu_group*)dist->emu_group;
          if (g->world != h->world) throw Fail{SCS_EINVAL, "emulated group size != world"};
          h->comm = new EmuComm(g, h->rank);
        } else if (dist->flags & SCS_DIST_HOST) {
          if (!dist->nccl_id || !dist->nccl_id[0])
            throw Fail{SCS_EINVAL, "host-shared-memory group needs its name in nccl_id"};
          char nm[129] = {0};
          memcpy(nm, dist->nccl_id, 128);
          h->comm = new ShmComm(nm, h->rank, h->world);
        } else {
#ifdef SCS_WITH_NCCL
          if (!dist->nccl_id) throw Fail{SCS_EINVAL, "row-sharded create needs an NCCL id"};
          NcclComm* nc = new NcclComm();
          h->comm = nc;
          ncclUniqueId id;
          memcpy(id.internal, dist->nccl_id, sizeof(id.internal));
          ncclResult_t r = ncclCommInitRank(&nc->c, h->world, id, h->rank);
          if (r != ncclSuccess)
            throw Fail{SCS_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)};
#else
          throw Fail{SCS_ENCCL, "built without NCCL"};
#endif
        }
        h->use_graph = h->comm->capturable();
      }
    } else if (P->row_lo != 0 || h->m_glob != m) {
      throw Fail{SCS_EINVAL, "a row slice needs a scs_dist"};
    }
    CK(cudaMallocHost((void**)&h->ctl_h, sizeof(Ctl)));
    CK(cudaMallocHost((void**)&h->loop_arg, sizeof(long long)));
    memset(h->ctl_h, 0, sizeof(Ctl));
    h->ctl = dalloc<Ctl>(h, 1);
    Ctl* c = h->ctl_h;
    c->alpha = S->alpha;
    c->cg_tol = (S->cg_tol > 0.0) ? S->cg_tol : 0.0;
    c->eps[0] = S->eps_pri; c->eps[1] = S->eps_dual; c->eps[2] = S->eps_gap;
    c->eps[3] = S->eps_infeas; c->eps[4] = S->eps_unbdd;
    c->max_iters = S->max_iters;
    c->check_interval = S->check_interval;
    c->status = SCS_RUNNING;
    c->denom = 1.0;
    c->sigma = c->rho = 1.0;
    push_ctl(h);
    dbg("ctl pushed");
    build_cones(h, P);
    dbg("cones built");
    // vectors
    Vec& V = h->V;
    V.n = n;
    V.m = m;
    V.ctl = h->ctl;
    V.u = dalloc<double>(h, n + m + 1);
    V.v = dalloc<double>(h, n + m + 1);
    h->b0 = dalloc<double>(h, m);
    h->c0 = dalloc<double>(h, n);
    h->bh = dalloc<double>(h, m);
    h->ch = dalloc<double>(h, n);
    h->D = dalloc<double>(h, m);
    h->E = dalloc<double>(h, n);
    V.c = h->ch; V.b = h->bh; V.D = h->D; V.E = h->E;
    V.gx = dalloc<double>(h, n);
    V.gy = dalloc<double>(h, m);
    V.rhs_x = dalloc<double>(h, n);
    V.x = dalloc<double>(h, n);
    V.r = dalloc<double>(h, n);
    V.Gp = dalloc<double>(h, n);
    V.X2 = dalloc<double>(h, 2 * n);
    V.P1 = dalloc<double>(h, n);
    V.Y2 = dalloc<double>(h, 2 * m);
    V.rhs_y = dalloc<double>(h, m);
    V.Axw = dalloc<double>(h, m);
    V.Aux = dalloc<double>(h, m);
    V.Agx = h->res_rec > 0 ? dalloc<double>(h, m) : nullptr;
    if (h->res_rec > 0 && h->res_rec_at) {
      V.T = dalloc<double>(h, n);
      V.AtAp = dalloc<double>(h, n);
      V.Sv = dalloc<double>(h, n);
      V.Uy = dalloc<double>(h, n);
      V.Dd = dalloc<double>(h, n);
      V.Atb = dalloc<double>(h, n);
      V.Atgy = dalloc<double>(h, n);
      V.Yc = dalloc<double>(h, m);
    }
    V.q = dalloc<double>(h, m);
    V.zy = dalloc<double>(h, m);
    V.Dinv = dalloc<double>(h, m);
    V.Einv = dalloc<double>(h, n);
    V.part = dalloc<double>(h, (size_t)kMaxRed * kMaxGrid);
    V.dred = dalloc<double>(h, kMaxRed);
    V.chunk_part = dalloc<double>(h, std::max(h->K.n_chunk, 1));
    V.soc_fac = dalloc<double>(h, 3 * std::max(h->K.n_bsoc, 1));
    V.cone_red = dalloc<double>(h, h->cone_red_len);
    if (getenv("SCS_DEBUG_PSD") && h->K.n_psd) {
      const size_t cap = 2 + (size_t)h->K.max_side * (h->K.max_side + 1) / 2;
      V.dbg = dalloc<double>(h, cap);
      CK(cudaMemsetAsync(V.dbg, 0, cap * sizeof(double), h->st));
    }
    V.xw = (!h->sharded || h->rank == 0) ? 1.0 : 0.0;
    if (h->sharded) h->Traw = dalloc<double>(h, 2 * std::max<long long>(n, 1));
    h->tmp_n = dalloc<double>(h, n);
    h->tmp_m = dalloc<double>(h, m);
    h->tmp_m2 = dalloc<double>(h, m);
    h->zero_m = dalloc<double>(h, m);
    h->dscal = dalloc<double>(h, 8);
    CK(cudaMemsetAsync(h->zero_m, 0, std::max<long long>(m, 1) * sizeof(double), h->st));
    h2d(h, h->b0, P->b, m);
    h2d(h, h->c0, P->c, n);
    dbg("create m=%lld n=%lld nnz=%lld", m, n, h->nnz);
    build_matrices(h, P);
    CK(cudaStreamSynchronize(h->st));
    dbg("matrices built LA=%d LAt=%d", h->LA, h->LAt);
    equilibrate(h);
    k_recip<<<elem_grid(h, m), kBlock, 0, h->st>>>(h->D, m, (double*)V.Dinv);
    k_recip<<<elem_grid(h, n), kBlock, 0, h->st>>>(h->E, n, (double*)V.Einv);
    dbg("equilibrated mean_col=%g mean_row=%g", h->mean_col, h->mean_row);
    setup_stream(h);
    dbg("streamed format built");
    setup_pcg(h);
    setup_split(h);
    scale_vectors(h);
    dbg("scaled sigma=%g rho=%g", h->sigma, h->rho);
    solve_g(h);
    dbg("g solved denom=%g cg=%lld", h->ctl_h->denom, h->ctl_h->cg_iters_total);
    build_graph(h);
    free_stage(h);
    dbg("graph built launches/iter=%lld", h->launches_per_iter);
    CK(cudaStreamSynchronize(h->st));
  });
  if (rc != SCS_OK) {
    h->err = scs_last_error(nullptr);
    scs_destroy(h);
    return rc;
  }
  h->setup_seconds = tm.s();
  *out = h;
  return SCS_OK;
}

int scs_begin(scs_handle* h, const double* wx, const double* wy, const double* ws) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] { do_begin(h, wx, wy, ws); });
}

int scs_step(scs_handle* h, int64_t k, scs_info* info) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] {
    do_steps(h, k);
    fill_info(h, info);
  });
}

int scs_finish(scs_handle* h, scs_info* info) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] {
    do_finish(h);
    fill_info(h, info);
  });
}

int scs_solve(scs_handle* h, const double* wx, const double* wy, const double* ws,
              scs_info* info) {
  if (!h) return SCS_EINVAL;
  Timer tm;
  return guard(h, [&] {
    do_begin(h, wx, wy, ws);
    do_steps(h, h->set.max_iters);
    do_finish(h);
    fill_info(h, info);
    if (info) info->solve_seconds = tm.s();
  });
}

int scs_get_state(scs_handle* h, double* u, double* v) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] {
    const long long len = h->n + h->m + 1;
    if (u) d2h(h, u, h->V.u, len);
    if (v) d2h(h, v, h->V.v, len);
    CK(cudaStreamSynchronize(h->st));
  });
}

int scs_get_scaling(scs_handle* h, double* D, double* E, double* sigma, double* rho) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] {
    if (D) d2h(h, D, h->D, h->m);
    if (E) d2h(h, E, h->E, h->n);
    CK(cudaStreamSynchronize(h->st));
    if (sigma) *sigma = h->sigma;
    if (rho) *rho = h->rho;
  });
}

int scs_update_vectors(scs_handle* h, const double* b, const double* c) {
  if (!h) return SCS_EINVAL;
  Timer tm;
  return guard(h, [&] {
    if (b) h2d(h, h->b0, b, h->m);
    if (c) h2d(h, h->c0, c, h->n);
    scale_vectors(h);
    solve_g(h);
    CK(cudaStreamSynchronize(h->st));
    h->setup_seconds = tm.s();
  });
}

int scs_apply_a(scs_handle* h, int which, const double* in, double* out) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] {
    const long long nin = which == 0 ? h->n : h->m, nout = which == 0 ? h->m : h->n;
    double* din = which == 0 ? h->tmp_n : h->tmp_m;
    double* dout = which == 0 ? h->tmp_m2 : h->V.Gp;
    h2d(h, din, in, nin);
    EpiPlain e{};
    e.V = h->V;
    e.xb = din;
    e.out = dout;
    if (which == 0) a_pass(h, e);
    else at_pass(h, e);
    d2h(h, out, dout, nout);
    CK(cudaStreamSynchronize(h->st));
  });
}

// _point_residuals (solver.py:237-248) of a device-resident point (dx: n,
// dy, ds: m; dx is also read after the passes).  out = {pri, dual, gap,
// c'x, b'y} (m-length sums all-reduced over row shards).
void point_residuals_dev(scs_handle* h, const double* dx, const double* dy, const double* ds,
                         double* out5, bool prod = false) {
  const long long n = h->n, m = h->m;
  const double* utau = h->V.u + n + m;
  // A x = D^-1 A_hat E^-1 x ; A^T y = E^-1 A_hat^T D^-1 y  (rows may be sharded:
  // m-length sums are all-reduced, A^T products go through at_pass).  With
  // `prod` (extraction of the final state), A_hat E^-1 x and A_hat^T D^-1 y
  // come from the products the last check kept (V.Aux, V.Uy): no matrix pass.
  if (prod) {
    k_prod_scale<<<elem_grid(h, m), kBlock, 0, h->st>>>(h->V.Aux, utau, h->sigma, m, h->tmp_m2);
  } else {
    k_div<<<elem_grid(h, n), kBlock, 0, h->st>>>(dx, h->E, n, h->V.r);
    EpiPlain e{};
    e.V = h->V;
    e.xb = h->V.r;
    e.out = h->tmp_m2;
    a_pass(h, e);
  }
  k_point_pri<<<elem_grid(h, m), kBlock, 0, h->st>>>(h->tmp_m2, h->D, ds, h->b0, m, h->V.q);
  const double pri = sqrt(norm2_dev(h, h->V.q, h->V.q, m, 2, true));
  const double bn = sqrt(norm2_dev(h, h->b0, h->b0, m, 2, true));
  if (prod) {
    k_prod_scale<<<elem_grid(h, n), kBlock, 0, h->st>>>(h->V.Uy, utau, h->rho, n, h->V.Gp);
  } else {
    k_div<<<elem_grid(h, m), kBlock, 0, h->st>>>(dy, h->D, m, h->tmp_m2);
    EpiPlain f{};
    f.V = h->V;
    f.xb = h->tmp_m2;
    f.out = h->V.Gp;
    at_pass(h, f);
  }
  k_point_dual<<<elem_grid(h, n), kBlock, 0, h->st>>>(h->V.Gp, h->E, h->c0, n, h->V.r);
  const double dual = sqrt(norm2_dev(h, h->V.r, h->V.r, n, 2));
  const double cn = sqrt(norm2_dev(h, h->c0, h->c0, n, 2));
  const double ctx = norm2_dev(h, h->c0, dx, n, 2);
  const double bty = norm2_dev(h, h->b0, dy, m, 2, true);
  out5[0] = pri / (1.0 + bn);
  out5[1] = dual / (1.0 + cn);
  out5[2] = fabs(ctx + bty) / (1.0 + fabs(ctx) + fabs(bty));
  out5[3] = ctx;
  out5[4] = bty;
}

double* ext_y(scs_handle* h) {
  if (!h->ext_y) h->ext_y = dalloc<double>(h, std::max<long long>(h->m, 1));
  return h->ext_y;
}

int scs_point_residuals(scs_handle* h, const double* x, const double* y, const double* s,
                        double* out3) {
  if (!h) return SCS_EINVAL;
  return guard(h, [&] {
    double* dy = ext_y(h);
    h2d(h, h->tmp_n, x, h->n);
    h2d(h, h->tmp_m, s, h->m);
    h2d(h, dy, y, h->m);
    double out5[5];
    point_residuals_dev(h, h->tmp_n, dy, h->tmp_m, out5);
    std::copy(out5, out5 + 3, out3);
  });
}

// extract_solution for a solved / max-iterations state (solver.py:251-270,
// scaling.py:140-145): x = E (u_x / tau) / sigma, y = D (u_y / tau) / rho,
// s = (v_s / tau) / (D sigma) formed on the device in the reference's
// operation order, copied out, and their point residuals computed from the
// device copies (no re-upload).
__global__ void k_extract(Vec V, const double* D, const double* E, double sigma, double rho,
                          double* x, double* y, double* s) {
  const long long n = V.n, m = V.m;
  const double ut = V.u[n + m];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < n + m; i += nt) {
    if (i < n) {
      x[i] = E[i] * (V.u[i] / ut) / sigma;
    } else {
      const long long j = i - n;
      y[j] = D[j] * (V.u[i] / ut) / rho;
      s[j] = (V.v[i] / ut) / (D[j] * sigma);
    }
  }
}

int scs_extract_point(scs_handle* h, double* x, double* y, double* s, double* out5) {
  if (!h || !out5) return SCS_EINVAL;
  return guard(h, [&] {
    double* dy = ext_y(h);
    k_extract<<<elem_grid(h, h->n + h->m), kBlock, 0, h->st>>>(h->V, h->D, h->E, h->sigma,
                                                                h->rho, h->tmp_n, dy, h->tmp_m);
    // the copies out run on a second stream, overlapped with the point
    // residuals (at full link speed when the caller's buffers are pinned)
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, h->st));
    CK(cudaStreamWaitEvent(h->st_copy, ev, 0));
    const long long n = h->n, m = h->m;
    if (x && n) CK(cudaMemcpyAsync(x, h->tmp_n, n * 8, cudaMemcpyDeviceToHost, h->st_copy));
    if (y && m) CK(cudaMemcpyAsync(y, dy, m * 8, cudaMemcpyDeviceToHost, h->st_copy));
    if (s && m) CK(cudaMemcpyAsync(s, h->tmp_m, m * 8, cudaMemcpyDeviceToHost, h->st_copy));
    // (tmp_n, dy, tmp_m are only read by the point residuals below)
    point_residuals_dev(h, h->tmp_n, dy, h->tmp_m, out5, h->prod_current);
    CK(cudaStreamSynchronize(h->st));
    CK(cudaStreamSynchronize(h->st_copy));
    cudaEventDestroy(ev);
  });
}

int scs_project_cone(int64_t z, int64_t l, int64_t nq, const int64_t* q, int64_t ns,
                     const int64_t* s, int64_t ep, int kind, int64_t n, const double* x,
                     double* out, int device) {
  scs_handle* h = new scs_handle();
  int rc = guard(nullptr, [&] {
    if (kind < 0 || kind > 2) throw Fail{SCS_EINVAL, "kind must be 0, 1 or 2"};
    h->dev = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->st_copy, cudaStreamNonBlocking));
    {
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, h->dev));
      unsigned long long keep = ~0ull;  // freed blocks stay in the pool (trimmed at destroy)
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device));
    h->grid_full = std::min(h->sms * (2048 / kBlock), kMaxGrid);
    long long m = z + l + 3 * ep;
    for (int64_t i = 0; i < nq; ++i) m += q[i];
    for (int64_t i = 0; i < ns; ++i) m += s[i] * (s[i] + 1) / 2;
    if (kind != 2) n = 0;
    h->m = h->m_glob = m;
    h->n = n;
    h->bounds = {0, m};
    scs_problem P{};
    P.m = m; P.n = n; P.z = z; P.l = l; P.nq = nq; P.q = q; P.ns = ns; P.s = s; P.ep = ep;
    build_cones(h, &P);
    CK(cudaMallocHost((void**)&h->ctl_h, sizeof(Ctl)));
    CK(cudaMallocHost((void**)&h->loop_arg, sizeof(long long)));
    memset(h->ctl_h, 0, sizeof(Ctl));
    h->ctl = dalloc<Ctl>(h, 1);
    Ctl* c = h->ctl_h;
    c->alpha = 1.0;
    c->corr = 0.0;
    c->check_interval = 1;
    c->status = SCS_RUNNING;
    push_ctl(h);
    const long long len = n + m + 1;
    std::vector<double> xin(len, 0.0);
    if (kind == 2) std::copy(x, x + len, xin.begin());
    else for (long long i = 0; i < m; ++i) xin[i] = kind == 1 ? -x[i] : x[i];
    Vec& V = h->V;
    V.n = n; V.m = m; V.ctl = h->ctl;
    V.u = dalloc<double>(h, len);
    V.v = dalloc<double>(h, len);
    V.x = dalloc<double>(h, n);
    V.gx = dalloc<double>(h, n);
    V.gy = dalloc<double>(h, m);
    V.zy = dalloc<double>(h, m);
    V.X2 = dalloc<double>(h, 2 * n);
    V.P1 = dalloc<double>(h, n);
    V.Y2 = dalloc<double>(h, 2 * m);
    double* zc = dalloc<double>(h, std::max<long long>(n, m));
    V.c = zc; V.b = zc;
    V.part = dalloc<double>(h, (size_t)kMaxRed * kMaxGrid);
    V.dred = dalloc<double>(h, kMaxRed);
    V.chunk_part = dalloc<double>(h, std::max(h->K.n_chunk, 1));
    V.soc_fac = dalloc<double>(h, 3 * std::max(h->K.n_bsoc, 1));
    V.cone_red = dalloc<double>(h, h->cone_red_len);
    V.xw = 1.0;
    CK(cudaMemsetAsync(zc, 0, std::max<long long>(n, m) * sizeof(double), h->st));
    CK(cudaMemsetAsync(V.gx, 0, std::max<long long>(n, 1) * sizeof(double), h->st));
    CK(cudaMemsetAsync(V.gy, 0, std::max<long long>(m, 1) * sizeof(double), h->st));
    CK(cudaMemsetAsync(V.u, 0, len * sizeof(double), h->st));
    CK(cudaMemsetAsync(V.v, 0, len * sizeof(double), h->st));
    h2d(h, V.x, xin.data(), n);
    h2d(h, V.zy, xin.data() + n, m);
    h2d(h, V.u + n + m, xin.data() + n + m, 1);  // u_tau = x_tau, v_tau = 0
    const long long work = std::max<long long>(n + h->K.z + h->K.l, 1);
    int g = std::max(elem_grid(h, work), std::min(h->K.n_chunk, h->grid_full));
    g = std::max(g, std::min((int)((h->K.n_ssoc * 32LL + kBlock - 1) / kBlock), h->grid_full));
    k_cone_tail<<<g, kBlock, 0, h->st>>>(V, h->K, 0);
    launch_cone_apply(h, V);
    CK(cudaGetLastError());
    std::vector<double> res(len);
    d2h(h, res.data(), V.u, len);
    pull_ctl(h);
    check_err(h);
    if (kind == 2) std::copy(res.begin(), res.end(), out);
    else if (kind == 0) std::copy(res.begin(), res.begin() + m, out);
    else for (long long i = 0; i < m; ++i) out[i] = x[i] + res[i];  // Pi_K(x) = x + Pi_K*(-x)
  });
  scs_destroy(h);
  return rc;
}

int scs_bench_iters(scs_handle* h, int64_t k, double* ms) {
  if (!h || !ms) return SCS_EINVAL;
  return guard(h, [&] {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const long long before = h->launches;
    CK(cudaEventRecord(e0, h->st));
    if (h->gloop) enqueue_loop(h, k);
    else for (int64_t i = 0; i < k; ++i) run_iteration(h);
    CK(cudaEventRecord(e1, h->st));
    CK(cudaEventSynchronize(e1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, e0, e1));
    *ms = f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    pull_ctl(h);
    if (h->gloop) account_loop(h);
    h->launches = h->launches - before;
    check_err(h);
  });
}

int scs_bench_kernel(scs_handle* h, int kind, int64_t reps, double* ms, double* bytes) {
  if (!h || !ms || !bytes) return SCS_EINVAL;
  return guard(h, [&] {
    pull_ctl(h);
    Ctl saved = *h->ctl_h;
    h->ctl_h->stop = 0;
    h->ctl_h->cg_done = 0;
    h->ctl_h->rs = 1.0;
    push_ctl(h);
    const long long m = h->m, n = h->n, nnz = h->nnz;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto one = [&] {
      if (kind == 0) {
        EpiAp<false> ea{};
        ea.V = h->V;
        ea.xb = h->V.P1;
        launch_mat(h, 0, ea);
      } else {
        EpiAtGp eg{};
        eg.V = h->V;
        eg.xb = h->V.q;
        at_pass(h, eg);
      }
    };
    one();
    CK(cudaEventRecord(e0, h->st));
    for (int64_t i = 0; i < reps; ++i) one();
    CK(cudaEventRecord(e1, h->st));
    CK(cudaEventSynchronize(e1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, e0, e1));
    *ms = f / (double)std::max<int64_t>(reps, 1);
    // algorithmic bytes: values + column indices, row pointers, the gathered
    // vector once, the epilogue vectors
    if (kind == 0) *bytes = 12.0 * nnz + 8.0 * (m + 1) + 8.0 * n + 8.0 * m;  // p gathered once
    else *bytes = 12.0 * nnz + 8.0 * (n + 1) + 8.0 * m + 16.0 * n;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *h->ctl_h = saved;
    push_ctl(h);
  });
}

int scs_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return SCS_EINVAL;
  *out = nullptr;
  const cudaError_t e = cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 8), cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_global_err(std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    return SCS_ENOMEM;
  }
  return SCS_OK;
}

void scs_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int scs_query(scs_handle* h, int32_t key, int64_t* out) {
  if (!h || !out) return SCS_EINVAL;
  switch (key) {
    case SCS_Q_FORMAT_A: *out = h->stm_m[0] ? 1 : 0; return SCS_OK;
    case SCS_Q_FORMAT_AT: *out = h->stm_m[1] ? 1 : 0; return SCS_OK;
    case SCS_Q_LAUNCHES_PER_ITER: *out = h->launches_per_iter; return SCS_OK;
    case SCS_Q_STREAM_BYTES_A: *out = (int64_t)h->stm_bytes[0]; return SCS_OK;
    case SCS_Q_STREAM_BYTES_AT: *out = (int64_t)h->stm_bytes[1]; return SCS_OK;
    case SCS_Q_CG_ITERS_TOTAL:
      return guard(h, [&] {
        pull_ctl(h);
        *out = h->ctl_h->cg_iters_total;
      });
    default: return SCS_EINVAL;
  }
}

int scs_allreduce(scs_handle* h, double* vals, int64_t n) {
  if (!h || n < 0 || n > 8) return SCS_EINVAL;
  return guard(h, [&] {
    h2d(h, h->dscal, vals, n);
    allreduce(h, h->dscal, n);
    d2h(h, vals, h->dscal, n);
    CK(cudaStreamSynchronize(h->st));
  });
}

int scs_nccl_unique_id(uint8_t* out128) {
#ifdef SCS_WITH_NCCL
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SCS_ENCCL;
  memcpy(out128, id.internal, 128);
  return SCS_OK;
#else
  (void)out128;
  set_global_err("built without NCCL");
  return SCS_ENCCL;
#endif
}

}  // extern "C"
