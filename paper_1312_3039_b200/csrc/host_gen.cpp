// host_gen.cpp -- host-side data producers around the hot path:
//   * scs_gen_lasso: sparse-F LASSO in gen_lasso's standard-form encoding
//     (reference generators.py:55-120) generated directly as CSC, in
//     parallel, for 1e8-1e9 nonzeros (the reference's dense
//     pure-Python generator cannot reach these sizes);
//   * scs_partition_rows: contiguous row shards for multi-GPU runs.
// Both are deterministic functions of their arguments, independent of the
// thread count (counter-based random streams per column / per row), and the
// generator is reproduced bit for bit by the pure-numpy
// generators.gen_lasso_hashed.  Compiled with -ffp-contract=off: every
// floating-point operation is a separately rounded IEEE +, * or sqrt.
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/scs_b200.h"

namespace {

// Counter-based streams: every random number is fmix64 of (stream base +
// counter), so the whole instance is a pure function of (seed, p, q, nnz_f)
// that numpy reproduces bit for bit (generators.gen_lasso_hashed: uint64
// wrap-around arithmetic, IEEE +,* only -- no libm -- so the CPU reference
// arm builds the same instance without this library).
inline uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
// stream base of object `j` in domain `dom` (0: F column rows, 1: F column
// values, 2: planted support keys, 3: planted values, 4: noise)
inline uint64_t base_of(uint64_t seed, uint64_t dom, uint64_t j) {
  return fmix64(seed * 0xD1B54A32D192ED03ull + dom * 0xA24BAED4963EE407ull + (j + 1) * kGold);
}
inline uint64_t draw(uint64_t base, uint64_t ctr) { return fmix64(base + (ctr + 1) * kGold); }
// Approximately N(0,1): Irwin-Hall sum of four 32-bit uniforms from two
// draws, centred and scaled to unit variance (exact IEEE operations in a
// fixed order).
inline double normal4(uint64_t base, uint64_t i) {
  const uint64_t a = draw(base, 2 * i), b = draw(base, 2 * i + 1);
  const double u1 = (double)(a >> 32) * 0x1p-32, u2 = (double)(a & 0xffffffffull) * 0x1p-32;
  const double u3 = (double)(b >> 32) * 0x1p-32, u4 = (double)(b & 0xffffffffull) * 0x1p-32;
  double s = u1 + u2;
  s = s + u3;
  s = s + u4;
  return (s - 2.0) * 1.7320508075688772;
}

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

// Column j of F: k sorted distinct rows of [0, q) with values normal4.
// Sparse columns (2k <= q): row_i = draw(i) mod q, sorted; every row equal
// to its predecessor is redrawn from counter (round << 32 | position) and
// the column re-sorted, until no duplicate is left.  Dense columns: the k
// rows with the smallest (key, row), key = draw(2^40 + row).
void f_column(uint64_t seed, int64_t j, int64_t k, int64_t q, std::vector<int64_t>& rows,
              std::vector<double>& vals) {
  const uint64_t br = base_of(seed, 0, (uint64_t)j), bv = base_of(seed, 1, (uint64_t)j);
  rows.resize(k);
  if (2 * k > q) {
    std::vector<std::pair<uint64_t, int64_t>> key(q);
    for (int64_t r = 0; r < q; ++r) key[r] = {draw(br, (1ull << 40) + (uint64_t)r), r};
    std::partial_sort(key.begin(), key.begin() + k, key.end());
    for (int64_t i = 0; i < k; ++i) rows[i] = key[i].second;
    std::sort(rows.begin(), rows.end());
  } else {
    for (int64_t i = 0; i < k; ++i) rows[i] = (int64_t)(draw(br, (uint64_t)i) % (uint64_t)q);
    std::sort(rows.begin(), rows.end());
    std::vector<int64_t> dup;
    for (uint64_t round = 1;; ++round) {
      dup.clear();  // positions equal to their predecessor, all found before any redraw
      for (int64_t i = 1; i < k; ++i)
        if (rows[i] == rows[i - 1]) dup.push_back(i);
      if (dup.empty()) break;
      for (int64_t i : dup) rows[i] = (int64_t)(draw(br, (round << 32) | (uint64_t)i) % (uint64_t)q);
      std::sort(rows.begin(), rows.end());
    }
  }
  vals.resize(k);
  for (int64_t i = 0; i < k; ++i) vals[i] = normal4(bv, (uint64_t)i);
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
  // planted coefficients (generators.py:72-75): p/10 support (the columns
  // with the smallest (key, column)), values normal4
  const int64_t ks = std::max<int64_t>(1, p / 10);
  std::vector<int64_t> support(ks);
  std::vector<double> zhat(ks);
  {
    std::vector<std::pair<uint64_t, int64_t>> key(p);
    const uint64_t bk = base_of(seed, 2, 0);
    for (int64_t j = 0; j < p; ++j) key[j] = {draw(bk, (uint64_t)j), j};
    std::partial_sort(key.begin(), key.begin() + ks, key.end());
    for (int64_t i = 0; i < ks; ++i) support[i] = key[i].second;
    std::sort(support.begin(), support.end());
    const uint64_t bz = base_of(seed, 3, 0);
    for (int64_t i = 0; i < ks; ++i) zhat[i] = normal4(bz, (uint64_t)i);
  }
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
      const uint64_t bn = base_of(seed, 4, 0);
      for (int64_t r = lo; r < hi; ++r) g[r] += normal4(bn, (uint64_t)r) * std::sqrt(0.1);
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
