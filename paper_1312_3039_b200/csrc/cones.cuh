// cones.cuh -- device projections for the cone blocks of K* (the y-part of
// the embedding iterate, cones.py:220-249):
//   zero block   -> free (identity)            cones.py:230-231
//   nonnegative  -> max(., 0)                  cones.py:232-233
//   SOC          -> three-branch formula       cones.py:172-184
//   PSD (svec)   -> eig-clamp via Jacobi       cones.py:147-191, _kernels.py:119-191
//   exponential  -> K_exp* = v + Pi_Kexp(-v)   (no reference)
#pragma once

#include "common.cuh"

namespace scs {

// ---------------------------------------------------------------------------
// exponential cone K_exp = cl{(r,s,t) : s > 0, s exp(r/s) <= t}
// Hard case: projection = s (rho, 1, e^rho) with polar part
// -lam (-1, rho-1, e^-rho); eliminating s and lam leaves the univariate root
//   F(rho) = ((rho-1) r0 + s0) e^rho - (r0 - rho s0) e^-rho
//            - t0 (rho^2 - rho + 1) = 0
// on the interval where s > 0 and lam > 0 (F is increasing there).  Solved
// by a safeguarded Newton iteration on an overflow-free rescaling of F with
// the same sign (the CPU oracle bisects instead: an independent check).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool exp_in_primal(double r, double s, double t) {
  return (s > 0.0 && s * exp(r / s) <= t) || (r <= 0.0 && s == 0.0 && t >= 0.0);
}
__device__ __forceinline__ bool exp_in_dual(double u, double v, double w) {
  return (u < 0.0 && -u * exp(v / u) <= 2.718281828459045 * w) ||
         (u == 0.0 && v >= 0.0 && w >= 0.0);
}

// G(rho) = F(rho) * q * e^{-rho} (rho >= 0) or F(rho) * q * e^{rho} (rho < 0),
// q = rho^2 - rho + 1 > 0: same sign as F, no overflow; and its derivative
// (for the Newton step).  With a = (rho-1) r0 + s0 (a' = r0),
// b = r0 - rho s0 (b' = -s0), q' = 2 rho - 1:
//   rho >= 0: G = a - b e^{-2rho} - t0 q e^{-rho},
//             G' = r0 + (s0 + 2b) e^{-2rho} - t0 (q' - q) e^{-rho}
//   rho <  0: G = a e^{2rho} - b - t0 q e^{rho},
//             G' = (r0 + 2a) e^{2rho} + s0 - t0 (q' + q) e^{rho}
__device__ __forceinline__ double exp_sign_fn(double rho, double r0, double s0, double t0,
                                              double* dG = nullptr) {
  const double q = rho * rho - rho + 1.0, dq = 2.0 * rho - 1.0;
  const double a = (rho - 1.0) * r0 + s0, b = r0 - rho * s0;
  if (rho >= 0.0) {
    const double e = exp(-rho), e2 = e * e;
    if (dG) *dG = r0 + (s0 + 2.0 * b) * e2 - t0 * (dq - q) * e;
    return a - b * e2 - t0 * q * e;
  }
  const double e = exp(rho), e2 = e * e;
  if (dG) *dG = (r0 + 2.0 * a) * e2 + s0 - t0 * (dq + q) * e;
  return a * e2 - b - t0 * q * e;
}

__device__ inline void exp_proj_primal(double r0, double s0, double t0, double* out) {
  if (exp_in_primal(r0, s0, t0)) { out[0] = r0; out[1] = s0; out[2] = t0; return; }
  if (exp_in_dual(-r0, -s0, -t0)) { out[0] = 0.0; out[1] = 0.0; out[2] = 0.0; return; }
  if (r0 <= 0.0 && s0 <= 0.0) { out[0] = r0; out[1] = 0.0; out[2] = fmax(t0, 0.0); return; }
  // root interval: s(rho) > 0 and lam(rho) > 0 (G increasing there)
  double lo = -INFINITY, hi = INFINITY;
  if (r0 > 0.0) lo = fmax(lo, 1.0 - s0 / r0);
  else if (r0 < 0.0) hi = fmin(hi, 1.0 - s0 / r0);
  if (s0 > 0.0) hi = fmin(hi, r0 / s0);
  else if (s0 < 0.0) lo = fmax(lo, r0 / s0);
  if (!isfinite(lo)) {
    lo = (isfinite(hi) ? hi : 0.0) - 1.0;
    for (int i = 0; i < 80 && exp_sign_fn(lo, r0, s0, t0) > 0.0; ++i) lo = 2.0 * lo - 1.0;
  }
  if (!isfinite(hi)) {
    hi = lo + 1.0;
    for (int i = 0; i < 80 && exp_sign_fn(hi, r0, s0, t0) < 0.0; ++i) hi = 2.0 * fabs(hi) + 1.0;
  }
  // safeguarded Newton: a Newton step from the current point when it lands
  // strictly inside the bracket, else bisection; the bracket shrinks with
  // the sign of G at every evaluated point (typically 4-8 evaluations)
  double rho = 0.5 * (lo + hi);
  for (int it = 0; it < 100; ++it) {
    double dG;
    const double G = exp_sign_fn(rho, r0, s0, t0, &dG);
    if (G == 0.0) { lo = hi = rho; break; }
    if (G < 0.0) lo = rho; else hi = rho;
    if (!(hi - lo > 1e-15 * fmax(1.0, fabs(rho)))) break;
    double nx = rho - G / dG;
    const bool newton = dG > 0.0 && nx > lo && nx < hi;
    if (!newton) nx = 0.5 * (lo + hi);
    if (nx <= lo || nx >= hi) break;
    if (newton && fabs(nx - rho) <= 1e-16 * fmax(1.0, fabs(rho))) { rho = nx; lo = hi = nx; break; }
    rho = nx;
  }
  rho = (lo == hi) ? lo : 0.5 * (lo + hi);
  const double q = rho * rho - rho + 1.0;
  const double s = ((rho - 1.0) * r0 + s0) / q;
  const double lam = (r0 - rho * s0) / q;
  out[0] = s * rho;
  out[1] = s;
  // t = s e^rho = t0 + lam e^-rho at the root; use the form that cannot blow up
  out[2] = rho > 0.0 ? t0 + lam * exp(-rho) : s * exp(rho);
}

// Pi_{K_exp*}(v) = v + Pi_{K_exp}(-v)  (Moreau)
__device__ __forceinline__ void exp_proj_dual(const double* v, double* out) {
  double p[3];
  exp_proj_primal(-v[0], -v[1], -v[2], p);
  out[0] = v[0] + p[0];
  out[1] = v[1] + p[1];
  out[2] = v[2] + p[2];
}

// ---------------------------------------------------------------------------
// PSD: packed column-major lower triangle with sqrt(2) off-diagonals
// (cones.py:23-64).  Element e of a side-k block -> (row, col).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void svec_rc(int e, int k, int& row, int& col) {
  int j = 0, start = 0;
  while (start + (k - j) <= e) { start += k - j; ++j; }
  col = j;
  row = j + (e - start);
}

// Round-robin (circle method) pairing for parallel cyclic Jacobi.
__device__ __forceinline__ int rr_player(int slot, int step, int kk) {
  return slot == 0 ? 0 : 1 + ((slot - 1 + step) % (kk - 1));
}

// Thread groups for the Jacobi eigensolver: a whole CTA (large blocks) or
// one warp (blocks of side <= kWarpPsd, many per CTA).
struct CtaGroup {
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return blockDim.x; }
  __device__ void sync() const { __syncthreads(); }
  __device__ double sum(double v) const {
    double a[1] = {v};
    block_sum<1>(a);
    return a[0];
  }
};
struct WarpGroup {
  __device__ int rank() const { return threadIdx.x & 31; }
  __device__ int size() const { return 32; }
  __device__ void sync() const { __syncwarp(); }
  __device__ double sum(double v) const { return warp_sum(v); }
};
constexpr int kWarpPsd = 16;  // sub-warp Jacobi up to this side (<= 8 pairs)

// Group-cooperative Jacobi eigensolve of the symmetric k x k matrix M
// (row-major, stride k) with eigenvectors V; same stopping rule as the
// reference (off-norm <= 1e-12 ||A||_F checked at sweep start, <= 100
// sweeps; _kernels.py:137-191).  The parallel (round-robin) rotation order
// differs from the reference's row-cyclic order; the projection it feeds is
// unique, so results agree to rounding.  Returns false on non-convergence.
// KC > 0: the side is a compile-time constant (warp path, sides <= 16), so
// the index arithmetic (/ k, % k, % (kk - 1)) folds to multiplies.
template <int KC, class G>
__device__ inline bool group_jacobi(const G& g, double* M, double* V, int k_rt, double* cs,
                                    double* sn, int* pp, int* qq, double* dpp, double* dqq) {
  const int k = KC > 0 ? KC : k_rt;
  const int tid = g.rank(), nt = g.size();
  for (int e = tid; e < k * k; e += nt) V[e] = (e / k == e % k) ? 1.0 : 0.0;
  double fro = 0.0;
  for (int e = tid; e < k * k; e += nt) fro += M[e] * M[e];
  fro = g.sum(fro);
  const double thresh = 1e-12 * sqrt(fro);
  // Entries below thresh / 2k are set to zero without a rotation: inside a
  // cluster of (near-)equal eigenvalues such entries are rounding noise, and
  // rotating by their arbitrary angles keeps moving the remaining coupling
  // between pairs, so the parallel ordering then converges only linearly
  // (seen on config 4 sector blocks: > 100 sweeps).  Dropping them perturbs
  // M by less than the stopping tolerance.
  const double tiny = thresh / (2.0 * k);
  if (k == 1) { g.sync(); return true; }
  const int kk = k + (k & 1);
  const int npair = kk / 2;
  for (int sweep = 0; sweep <= 100; ++sweep) {
    double off = 0.0;
    for (int e = tid; e < k * k; e += nt) {
      const int i = e / k, j = e % k;
      if (j > i) off += 2.0 * M[e] * M[e];
    }
    off = g.sum(off);
    if (sqrt(off) <= thresh) return true;
    if (sweep == 100) return false;
    for (int step = 0; step < kk - 1; ++step) {
      for (int pi = tid; pi < npair; pi += nt) {
        int a = rr_player(pi, step, kk), b = rr_player(kk - 1 - pi, step, kk);
        int p = a < b ? a : b, q = a < b ? b : a;
        double c = 1.0, s = 0.0, np = 0.0, nq = 0.0;
        if (q < k) {
          const double apq = M[p * k + q];
          const double app = M[p * k + p], aqq = M[q * k + q];
          np = app; nq = aqq;
          if (fabs(apq) > tiny) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double root = sqrt(1.0 + tau * tau);
            const double t = tau >= 0.0 ? 1.0 / (tau + root) : 1.0 / (tau - root);
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            np = app - t * apq;
            nq = aqq + t * apq;
          }
        } else {
          p = -1;  // dummy pairing for odd k
        }
        pp[pi] = p; qq[pi] = q; cs[pi] = c; sn[pi] = s; dpp[pi] = np; dqq[pi] = nq;
      }
      g.sync();
      // M <- M J (columns p, q)
      for (int w = tid; w < npair * k; w += nt) {
        const int pi = w / k, i = w % k, p = pp[pi];
        if (p < 0 || sn[pi] == 0.0) continue;
        const int q = qq[pi];
        const double a = M[i * k + p], b = M[i * k + q];
        M[i * k + p] = cs[pi] * a - sn[pi] * b;
        M[i * k + q] = sn[pi] * a + cs[pi] * b;
      }
      g.sync();
      // M <- J^T M (rows p, q) and V <- V J
      for (int w = tid; w < npair * k; w += nt) {
        const int pi = w / k, j = w % k, p = pp[pi];
        if (p < 0 || sn[pi] == 0.0) continue;
        const int q = qq[pi];
        const double a = M[p * k + j], b = M[q * k + j];
        M[p * k + j] = cs[pi] * a - sn[pi] * b;
        M[q * k + j] = sn[pi] * a + cs[pi] * b;
        const double va = V[j * k + p], vb = V[j * k + q];
        V[j * k + p] = cs[pi] * va - sn[pi] * vb;
        V[j * k + q] = sn[pi] * va + cs[pi] * vb;
      }
      g.sync();
      for (int pi = tid; pi < npair; pi += nt) {
        const int p = pp[pi];
        if (p < 0) continue;
        const int q = qq[pi];
        if (sn[pi] != 0.0) {
          M[p * k + p] = dpp[pi];
          M[q * k + q] = dqq[pi];
        }
        M[p * k + q] = 0.0;
        M[q * k + p] = 0.0;
      }
      g.sync();
    }
  }
  return false;
}

__device__ inline bool block_jacobi(double* M, double* V, int k, double* cs, double* sn, int* pp,
                                    int* qq, double* dpp, double* dqq) {
  return group_jacobi<0>(CtaGroup{}, M, V, k, cs, sn, pp, qq, dpp, dqq);
}

}  // namespace scs
