// stm_sim.cpp -- host model of the streamed-tile format (stream.cuh): builds
// warp sections with the same pin/overflow/bank-balancing rules as k_stm_pin
// on synthetic C5-like sections and counts shared-memory wavefronts per
// entry (values, slot words, gathers, accumulator read-modify-writes) and
// slots per entry (padding).  Used to choose format parameters before
// spending GPU time.  g++ -O2 -o /tmp/stm_sim tools/stm_sim.cpp
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <random>
#include <vector>

constexpr int kPinMax = 128;

struct Ent { uint64_t key; int perm; };

// returns D (0 = fail); fills slot[] (step*32+lane | ovf<<30), hown[32]
int pin(std::vector<uint64_t>& key, std::vector<int>& slot, int* hown_out, int partner_pref) {
  const long long p0 = 0, p1 = key.size();
  const long long E = p1 - p0;
  for (int l = 0; l < 32; ++l) hown_out[l] = 0xff;
  if (E == 0) return 0;
  const int D0 = (int)((E + 31) / 32);
  int cnt[32], host[32];
  long long run0[32];
  unsigned freem[kPinMax];
  int ostep[kPinMax];
  for (int l = 0; l < 32; ++l) cnt[l] = 0;
  for (long long e = p0; e < p1; ++e) cnt[(key[e] >> 7) & 31u]++;
  { long long r = p0; for (int l = 0; l < 32; ++l) { run0[l] = r; r += cnt[l]; } }
  bool ok = false;
  int D = D0;
  std::vector<int> perm(E);
  for (int i = 0; i < E; ++i) perm[i] = i;
  for (; !ok && D <= 2 * D0 + 16 && D <= kPinMax; ++D) {
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
    for (int l = 0; l < 32; ++l) host[l] = -1;
    for (int g = 0; g < 32 && ok; ++g) {
      int l = -1, o = 0;
      for (int c = 0; c < 32; ++c)
        if (!(done >> c & 1u) && cnt[c] - D > o) { o = cnt[c] - D; l = c; }
      if (l < 0) break;
      done |= 1u << l;
      unsigned allow = 0;
      for (int c = 0; c < 32; ++c)
        if (c != l && (host[c] < 0 || host[c] == l)) allow |= 1u << c;
      if (partner_pref == 2) allow &= 1u << (l ^ 16);  // strict: partner lane only
      const unsigned partner = partner_pref ? ((1u << (l ^ 16)) & allow) : 0u;
      int n = 0;
      for (int k = D - 1; k >= 0 && n < o; --k)
        if (freem[k] & partner) ostep[n++] = k;
      for (int k = D - 1; k >= 0 && n < o; --k)
        if ((freem[k] & allow) && !(freem[k] & partner)) ostep[n++] = k;
      if (n < o) { ok = false; break; }
      const long long run = run0[l];
      for (int q = 0; q < o && ok; ++q) {
        const long long a = run + ostep[q], b = run + D + q;
        const unsigned jb = (unsigned)(key[b] & 7u);
        if ((unsigned)(key[a] & 7u) != jb) continue;
        bool fixed = false;
        for (int k2 = 0; k2 < D && !fixed; ++k2) {
          const long long c2 = run + k2;
          if ((unsigned)(key[c2] & 7u) == jb) continue;
          int q2 = -1;
          for (int t = 0; t < o; ++t) if (ostep[t] == k2) q2 = t;
          if (q2 >= 0 && (unsigned)(key[run + D + q2] & 7u) == jb) continue;
          std::swap(key[a], key[c2]);
          fixed = true;
        }
        ok = fixed;
      }
      for (int q = 0; q < o && ok; ++q) {
        const int k = ostep[q];
        const unsigned m = freem[k] & allow;
        int lane = -1;
        if (m & partner) lane = l ^ 16;
        for (int c = 0; c < 32 && lane < 0; ++c)
          if ((m >> c & 1u) && host[c] == l) lane = c;
        if (lane < 0) lane = __builtin_ffs(m) - 1;
        host[lane] = l;
        freem[k] &= ~(1u << lane);
        slot[run + D + q] = (k * 32 + lane) | (1 << 30);
      }
    }
    if (ok) {
      static unsigned char use[kPinMax][2][16], useq[kPinMax][4][8];
      for (int k = 0; k < D; ++k) {
        for (int h = 0; h < 2; ++h) for (int b = 0; b < 16; ++b) use[k][h][b] = 0;
        for (int h = 0; h < 4; ++h) for (int b = 0; b < 8; ++b) useq[k][h][b] = 0;
      }
      auto bank = [&](long long e) { return (unsigned)(((key[e] >> 3) + (key[e] >> 7)) & 15u); };
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
          const long long e_end = run0[l] + (cnt[l] < i + 8 ? cnt[l] : i + 8);
          for (long long e = run0[l] + i; e < e_end; ++e) {
            const unsigned b = bank(e);
            const int u = 4 * useq[k][l >> 3][b & 7u] + use[k][l >> 4][b];
            if (u < bu) { bu = u; best = e; }
          }
          const long long a = run0[l] + i;
          if (best != a) std::swap(key[a], key[best]);
          use[k][l >> 4][bank(a)]++;
          useq[k][l >> 3][bank(a) & 7u]++;
          slot[a] = k * 32 + l;
        }
      }
    }
  }
  if (!ok) return 0;
  for (int l = 0; l < 32; ++l) hown_out[l] = host[l];
  return D - 1;
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 2048;
  const double E_mean = argc > 2 ? atof(argv[2]) : 116.0;  // entries per 256-row section
  const int nsec = argc > 3 ? atoi(argv[3]) : 3000;
  const int partner = argc > 4 ? atoi(argv[4]) : 1;
  const int search = argc > 5 ? atoi(argv[5]) : 0;
  const int search_ovf = argc > 6 ? atoi(argv[6]) : 0;
  std::mt19937_64 rng(1);
  std::poisson_distribution<int> pois(E_mean);
  double slots = 0, ents = 0, wf_g = 0, wf_r = 0, steps = 0, fails = 0;
  for (int s = 0; s < nsec; ++s) {
    const int E = pois(rng);
    std::vector<uint64_t> key(E);
    std::vector<int> col(E);
    for (int e = 0; e < E; ++e) {
      const unsigned rl = rng() % 256, c = rng() % W, ln = rl & 31;
      const unsigned bank = (c - ln) & 15u;
      // key low bits: lane << 7 | bank << 3 | j ; keep the column beside it
      key[e] = ((uint64_t)c << 12) | (ln << 7) | (bank << 3) | (rl >> 5);
    }
    std::sort(key.begin(), key.end(), [](uint64_t a, uint64_t b) { return (a & 0xfff) < (b & 0xfff) || ((a & 0xfff) == (b & 0xfff) && a < b); });
    std::vector<int> slot(E, -1);
    int hown[32];
    const int D = pin(key, slot, hown, partner);
    if (D <= 0) { fails++; continue; }
    // grid of (step, lane) -> entry
    std::vector<long long> grid(D * 32, -1);
    for (int e = 0; e < E; ++e) grid[slot[e] & ((1 << 30) - 1)] = e;
    auto colof = [&](long long e, int l) { return e < 0 ? l : (int)(key[e] >> 12); };
    auto rowof = [&](long long e, int l) -> int {
      if (e < 0) return -1;
      const int j = key[e] & 7, ovf = slot[e] >> 30;
      return j * 32 + (ovf ? hown[l] : l);
    };
    // cost of one (step, half): gather max-class distinct cols + 2 x RMW max-class distinct rows
    auto cost = [&](int k, int h) {
      int gb[16][32], gn[16] = {}, rb[16][32], rn[16] = {};
      for (int l = h * 16; l < h * 16 + 16; ++l) {
        const long long e = grid[k * 32 + l];
        const int c = colof(e, l), row = rowof(e, l);
        bool seen = false;
        for (int t = 0; t < gn[c & 15]; ++t) seen |= gb[c & 15][t] == c;
        if (!seen) gb[c & 15][gn[c & 15]++] = c;
        if (row >= 0) {
          bool s2 = false;
          for (int t = 0; t < rn[row & 15]; ++t) s2 |= rb[row & 15][t] == row;
          if (!s2) rb[row & 15][rn[row & 15]++] = row;
        }
      }
      int mg = 0, mr = 0;
      for (int b = 0; b < 16; ++b) { mg = std::max(mg, gn[b]); mr = std::max(mr, rn[b]); }
      return mg + 2 * mr;
    };
    if (search < 0) {  // simulated annealing over within-lane step swaps (same constraints)
      std::mt19937 r2(s + 7);
      auto conflict2 = [&](long long e, int k, int l) {
        if (e < 0) return false;
        const int rr = rowof(e, l);
        for (int c = 0; c < 32; ++c) {
          if (c == l) continue;
          const long long f = grid[k * 32 + c];
          if (f >= 0 && rowof(f, c) == rr) return true;
        }
        return false;
      };
      const int iters = -search * 32 * D * D;
      double T = 2.0;
      for (int it = 0; it < iters; ++it, T *= 0.9995) {
        const int l = r2() % 32, k1 = r2() % D, k2 = r2() % D;
        if (k1 == k2) continue;
        long long& a = grid[k1 * 32 + l];
        long long& b = grid[k2 * 32 + l];
        if (a < 0 && b < 0) continue;
        if (conflict2(a, k2, l) || conflict2(b, k1, l)) continue;
        const int h = l >> 4;
        const int before = cost(k1, h) + cost(k2, h);
        std::swap(a, b);
        const int after = cost(k1, h) + cost(k2, h);
        const int dlt = after - before;
        if (dlt > 0 && std::uniform_real_distribution<double>(0, 1)(r2) >= std::exp(-dlt / T)) std::swap(a, b);
      }
    }
    if (search > 0) {
      // local search: swap two steps' contents within one lane (pinned entries
      // and padding only), keeping no step with a pinned and an overflow entry
      // of the same row
      auto conflict = [&](long long e, int k, int l) {  // e (of lane l) placed at step k: rows distinct?
        if (e < 0) return false;
        const int r = rowof(e, l);
        for (int c = 0; c < 32; ++c) {
          if (c == l) continue;
          const long long f = grid[k * 32 + c];
          if (f >= 0 && rowof(f, c) == r) return true;
        }
        return false;
      };
      for (int pass = 0; pass < search; ++pass) {
        bool any = false;
        for (int l = 0; l < 32; ++l)
          for (int k1 = 0; k1 < D; ++k1)
            for (int k2 = k1 + 1; k2 < D; ++k2) {
              long long& a = grid[k1 * 32 + l];
              long long& b = grid[k2 * 32 + l];
              if (search_ovf == 0 && ((a >= 0 && (slot[a] >> 30)) || (b >= 0 && (slot[b] >> 30)))) continue;
              if (a < 0 && b < 0) continue;
              if (conflict(a, k2, l) || conflict(b, k1, l)) continue;
              const int h = l >> 4;
              const int before = cost(k1, h) + cost(k2, h);
              std::swap(a, b);
              const int after = cost(k1, h) + cost(k2, h);
              if (after < before) any = true;
              else std::swap(a, b);
            }
        if (!any) break;
      }
    }
    for (int k = 0; k < D; ++k) {
      for (int h = 0; h < 2; ++h) {
        int gb[16][64] = {}, gn[16] = {};
        int rb[16][64] = {}, rn[16] = {};
        for (int l = h * 16; l < h * 16 + 16; ++l) {
          const long long e = grid[k * 32 + l];
          int c, row = -1;
          if (e < 0) c = l;  // padding gathers column = lane
          else {
            c = (int)(key[e] >> 12);
            const int j = key[e] & 7, ovf = slot[e] >> 30;
            const int ownlane = ovf ? hown[l] : l;
            row = j * 32 + ownlane;
          }
          const int gbk = c & 15;
          bool seen = false;
          for (int t = 0; t < gn[gbk]; ++t) seen |= gb[gbk][t] == c;
          if (!seen) gb[gbk][gn[gbk]++] = c;
          if (row >= 0) {
            const int rbk = row & 15;
            bool s2 = false;
            for (int t = 0; t < rn[rbk]; ++t) s2 |= rb[rbk][t] == row;
            if (!s2) rb[rbk][rn[rbk]++] = row;
          }
        }
        int mg = 0, mr = 0;
        for (int b = 0; b < 16; ++b) { mg = std::max(mg, gn[b]); mr = std::max(mr, rn[b]); }
        wf_g += mg;
        wf_r += mr;
      }
      steps += 1;
    }
    slots += 32.0 * D;
    ents += E;
  }
  const double per32 = 32.0 / ents;
  const double tot = wf_g * per32 + 2 * wf_r * per32 + 3 * steps * per32 + (10.0 * slots / ents) * 32 / 128 + 2.2;
  printf("search=%d W=%d E=%.0f partner=%d: slots/entry %.3f  steps/32ent %.3f | per 32 entries: gather %.2f  acc(rd) %.2f  vals %.2f idx %.2f  fails %.0f  TOTAL %.2f\n",
         search, W, E_mean, partner, slots / ents, steps * per32, wf_g * per32, wf_r * per32, 2 * steps * per32,
         steps * per32, fails, tot);
  return 0;
}
