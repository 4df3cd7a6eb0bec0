// host_gen.cpp -- host-side data producers around the hot path:
//   * scs_gen_lasso: sparse-F LASSO in gen_lasso's standard-form encoding
//     (reference generators.py:55-120) generated directly as CSC, in
//     parallel, for 1e8-1e9 nonzeros (the reference's dense
//     pure-Python generator cannot reach these sizes);
//   * scs_partition_rows: contiguous row shards for multi-GPU runs.
// Both are deterministic functions of their arguments, independent of the
// thread count (counter-based random streams per column / per row).
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/scs_b200.h"

namespace {

inline uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// xoshiro256** seeded by splitmix64 (the family of reference rng.py:16-50;
// not bit-compatible with it, which the reference does not promise either)
struct Rng {
  uint64_t s[4];
  bool has_spare = false;
  double spare = 0.0;
  explicit Rng(uint64_t seed) {
    for (auto& w : s) w = splitmix(seed);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return (next() >> 11) * 0x1.0p-53; }
  double normal() {  // Box-Muller (rng.py:59-70)
    if (has_spare) { has_spare = false; return spare; }
    const double u1 = 1.0 - uniform(), u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1)), th = 6.283185307179586 * u2;
    spare = r * std::sin(th);
    has_spare = true;
    return r * std::cos(th);
  }
  uint64_t below(uint64_t n) {  // unbiased (rng.py:75-83)
    const uint64_t lim = UINT64_MAX - (UINT64_MAX % n);
    for (;;) {
      const uint64_t u = next();
      if (u < lim) return u % n;
    }
  }
};

template <class F>
void parallel_for(int64_t n, int threads, F&& fn) {
  if (threads <= 1 || n < 2) {
    for (int64_t i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (;;) {
        const int64_t i0 = next.fetch_add(64);
        if (i0 >= n) break;
        const int64_t i1 = std::min<int64_t>(n, i0 + 64);
        for (int64_t i = i0; i < i1; ++i) fn(i, t);
      }
    });
  for (auto& th : pool) th.join();
}

// Column j of F: k sorted distinct rows of [0, q) with N(0,1) values.
void f_column(uint64_t seed, int64_t j, int64_t k, int64_t q, std::vector<int64_t>& rows,
              std::vector<double>& vals) {
  Rng rng(seed ^ (0xA24BAED4963EE407ull * (uint64_t)(j + 1)));
  rows.resize(k);
  if (2 * k > q) {  // selection sampling (Knuth S)
    int64_t need = k, t = 0;
    for (int64_t r = 0; r < q && need; ++r)
      if ((double)(q - r) * rng.uniform() < (double)need) { rows[t++] = r; --need; }
  } else {
    for (int64_t i = 0; i < k; ++i) rows[i] = (int64_t)rng.below(q);
    std::sort(rows.begin(), rows.end());
    for (int round = 0; round < 64; ++round) {
      int64_t dup = 0;
      for (int64_t i = 1; i < k; ++i)
        if (rows[i] == rows[i - 1]) { rows[i] = (int64_t)rng.below(q); ++dup; }
      if (!dup) break;
      std::sort(rows.begin(), rows.end());
    }
  }
  vals.resize(k);
  for (int64_t i = 0; i < k; ++i) vals[i] = rng.normal();
}

}  // namespace

extern "C" int scs_gen_lasso(int64_t p, int64_t q, int64_t nnz_f, uint64_t seed, int64_t row_lo,
                             int64_t row_hi, int threads, int64_t* m_out, int64_t* n_out,
                             int64_t* nnz_out, int64_t* colptr, int64_t* rowidx, double* vals,
                             double* b, double* c) {
  if (p < 1 || q < 1 || nnz_f < 0 || nnz_f > p * q) return SCS_EINVAL;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t n = 2 * p + 1, m = 2 * p + q + 2;  // generators.py:81-82
  if (row_hi <= 0 || row_hi > m) row_hi = m;
  if (row_lo < 0 || row_lo > row_hi) return SCS_EINVAL;
  const int64_t r0 = 2 * p;  // first SOC row
  auto kcol = [&](int64_t j) { return nnz_f / p + (j < nnz_f % p ? 1 : 0); };
  auto in = [&](int64_t r) { return r >= row_lo && r < row_hi; };
  // structural counts per column for the slice
  std::vector<int64_t> cnt(n, 0);
  parallel_for(p, threads, [&](int64_t j, int) {
    std::vector<int64_t> rows;
    std::vector<double> vv;
    int64_t k = in(j) + in(p + j);
    // count F rows in [row_lo - r0 - 2, row_hi - r0 - 2)
    const int64_t flo = row_lo - r0 - 2, fhi = row_hi - r0 - 2;
    if (fhi > 0 && flo < q) {
      f_column(seed, j, kcol(j), q, rows, vv);
      k += std::lower_bound(rows.begin(), rows.end(), fhi) -
           std::lower_bound(rows.begin(), rows.end(), flo);
    }
    cnt[j] = k;
    cnt[p + j] = in(j) + in(p + j);
  });
  cnt[2 * p] = in(r0) + in(r0 + 1);
  int64_t nnz = 0;
  for (int64_t j = 0; j < n; ++j) nnz += cnt[j];
  if (m_out) *m_out = row_hi - row_lo;
  if (n_out) *n_out = n;
  if (nnz_out) *nnz_out = nnz;
  if (!colptr) return SCS_OK;
  colptr[0] = 0;
  for (int64_t j = 0; j < n; ++j) colptr[j + 1] = colptr[j] + cnt[j];
  // planted coefficients (generators.py:72-75): p/10 support, N(0,1)
  Rng grng(seed * 0x9E3779B97F4A7C15ull + 17);
  const int64_t ks = std::max<int64_t>(1, p / 10);
  std::vector<int64_t> pool(p);
  for (int64_t i = 0; i < p; ++i) pool[i] = i;
  for (int64_t i = 0; i < ks; ++i) std::swap(pool[i], pool[i + (int64_t)grng.below(p - i)]);
  std::vector<int64_t> support(pool.begin(), pool.begin() + ks);
  std::sort(support.begin(), support.end());
  std::vector<double> zhat(ks);
  for (int64_t i = 0; i < ks; ++i) zhat[i] = grng.normal();
  std::vector<int64_t>().swap(pool);
  // g = F zhat + sqrt(0.1) noise (generators.py:76-77); deterministic by
  // accumulating each row block over the support columns in order
  std::vector<double> g(q, 0.0);
  {
    std::vector<std::vector<int64_t>> srows(ks);
    std::vector<std::vector<double>> svals(ks);
    parallel_for(ks, threads, [&](int64_t i, int) {
      f_column(seed, support[i], kcol(support[i]), q, srows[i], svals[i]);
    });
    const int64_t nb = std::max<int64_t>(1, threads * 4);
    parallel_for(nb, threads, [&](int64_t blk, int) {
      const int64_t lo = q * blk / nb, hi = q * (blk + 1) / nb;
      for (int64_t i = 0; i < ks; ++i) {
        auto& R = srows[i];
        auto it = std::lower_bound(R.begin(), R.end(), lo);
        for (int64_t e = it - R.begin(); e < (int64_t)R.size() && R[e] < hi; ++e)
          g[R[e]] += svals[i][e] * zhat[i];
      }
      for (int64_t r = lo; r < hi; ++r) {
        Rng nr(seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(r + 1)));
        g[r] += nr.normal() * std::sqrt(0.1);
      }
    });
  }
  // mu = 0.1 ||F^T g||_inf (generators.py:78-79)
  std::vector<double> ftg(p, 0.0);
  parallel_for(p, threads, [&](int64_t j, int) {
    std::vector<int64_t> rows;
    std::vector<double> vv;
    f_column(seed, j, kcol(j), q, rows, vv);
    double s = 0.0;
    for (size_t e = 0; e < rows.size(); ++e) s += vv[e] * g[rows[e]];
    ftg[j] = std::fabs(s);
  });
  double mu = 0.0;
  for (double v : ftg) mu = std::max(mu, v);
  mu *= 0.1;
  // fill CSC of the slice (generators.py:86-118), local row indices
  parallel_for(p, threads, [&](int64_t j, int) {
    int64_t o = colptr[j];
    if (in(j)) { rowidx[o] = j - row_lo; vals[o] = 1.0; ++o; }
    if (in(p + j)) { rowidx[o] = p + j - row_lo; vals[o] = -1.0; ++o; }
    const int64_t flo = row_lo - r0 - 2, fhi = row_hi - r0 - 2;
    if (fhi > 0 && flo < q) {
      std::vector<int64_t> rows;
      std::vector<double> vv;
      f_column(seed, j, kcol(j), q, rows, vv);
      for (size_t e = 0; e < rows.size(); ++e)
        if (rows[e] >= flo && rows[e] < fhi) {
          rowidx[o] = r0 + 2 + rows[e] - row_lo;
          vals[o] = 2.0 * vv[e];
          ++o;
        }
    }
    int64_t o2 = colptr[p + j];
    if (in(j)) { rowidx[o2] = j - row_lo; vals[o2] = -1.0; ++o2; }
    if (in(p + j)) { rowidx[o2] = p + j - row_lo; vals[o2] = -1.0; ++o2; }
  });
  {
    int64_t o = colptr[2 * p];
    if (in(r0)) { rowidx[o] = r0 - row_lo; vals[o] = -1.0; ++o; }
    if (in(r0 + 1)) { rowidx[o] = r0 + 1 - row_lo; vals[o] = 1.0; ++o; }
  }
  if (b) {
    for (int64_t r = row_lo; r < row_hi; ++r) {
      double v = 0.0;
      if (r == r0 || r == r0 + 1) v = 1.0;
      else if (r >= r0 + 2) v = 2.0 * g[r - r0 - 2];
      b[r - row_lo] = v;
    }
  }
  if (c) {
    for (int64_t j = 0; j < p; ++j) { c[j] = 0.0; c[p + j] = mu; }
    c[2 * p] = 0.5;
  }
  return SCS_OK;
}

// Contiguous row shards.  Allowed cut points: anywhere in the zero/nonneg
// rows, anywhere inside a second-order cone (its norm is all-reduced),
// never strictly inside a PSD or exponential block.  Cuts are placed where
// the running weight (nnz per row) crosses k * total / world.
extern "C" int scs_partition_rows(int64_t z, int64_t l, int64_t nq, const int64_t* q, int64_t ns,
                                  const int64_t* s, int64_t ep, const int64_t* row_nnz,
                                  int32_t world, int64_t* bounds) {
  if (world < 1) return SCS_EINVAL;
  int64_t m = z + l;
  for (int64_t i = 0; i < nq; ++i) m += q[i];
  const int64_t soc_end = m;
  std::vector<std::pair<int64_t, int64_t>> rigid;  // [lo, hi) blocks that cannot be cut
  for (int64_t i = 0; i < ns; ++i) {
    const int64_t d = s[i] * (s[i] + 1) / 2;
    rigid.push_back({m, m + d});
    m += d;
  }
  for (int64_t i = 0; i < ep; ++i) { rigid.push_back({m, m + 3}); m += 3; }
  (void)soc_end;
  std::vector<int64_t> cum(m + 1, 0);
  for (int64_t r = 0; r < m; ++r) cum[r + 1] = cum[r] + (row_nnz ? row_nnz[r] : 1) + 1;
  bounds[0] = 0;
  bounds[world] = m;
  for (int32_t k = 1; k < world; ++k) {
    const double target = (double)cum[m] * k / world;
    int64_t r = std::lower_bound(cum.begin(), cum.end(), (int64_t)std::ceil(target)) - cum.begin();
    r = std::min<int64_t>(std::max<int64_t>(r, bounds[k - 1]), m);
    // move out of a rigid block to its nearest end
    auto it = std::upper_bound(rigid.begin(), rigid.end(), std::make_pair(r, INT64_MAX));
    if (it != rigid.begin()) {
      --it;
      if (r > it->first && r < it->second) r = (r - it->first <= it->second - r) ? it->first : it->second;
    }
    bounds[k] = std::max<int64_t>(r, bounds[k - 1]);
  }
  return SCS_OK;
}
