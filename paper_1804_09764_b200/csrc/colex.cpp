// colex.cpp -- colour-set indexing with the combinatorial number system and
// the split / lift / complement tables of the DP steps.
//
// PAPER.md Alg. 1 line 8 (lines 159-160): "for v in V, T_i in T and subset
// S_i subset of S with |S_i| = |T_i|" -- every table row holds C(k, |T_i|)
// entries, one per colour set; Eq. 1/2 (lines 118, 167) sum over the splits
// S = S1 u S2 with |S1| = |T_i'|, |S2| = |T_i''|.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.h"

namespace cc {

int64_t binom(int n, int r) {
  if (r < 0 || n < 0 || r > n) return 0;
  int64_t c = 1;
  for (int i = 1; i <= r; ++i) c = c * (n - r + i) / i;
  return c;
}

// rank(S) = sum_i C(s_i, i + 1) over the elements s_0 < s_1 < ... of S.
int64_t colex_rank(uint32_t mask) {
  int64_t r = 0;
  int i = 0;
  for (int c = 0; c < 32; ++c)
    if (mask >> c & 1u) r += binom(c, ++i);
  return r;
}

uint32_t colex_unrank(int s, int64_t r) {
  if (s < 0 || s > kMaxK || r < 0) return 0xFFFFFFFFu;
  uint32_t mask = 0;
  int hi = 31;
  for (int i = s; i >= 1; --i) {
    // largest c with C(c, i) <= r
    int c = i - 1;
    while (c + 1 <= hi && binom(c + 1, i) <= r) ++c;
    r -= binom(c, i);
    mask |= 1u << c;
    hi = c - 1;
  }
  return r == 0 ? mask : 0xFFFFFFFFu;
}

std::vector<uint32_t> split_table(int k, int t, int a) {
  const int64_t nS = binom(k, t), nq = binom(t, a);
  std::vector<uint32_t> out((size_t)(nS * nq));
  int elem[kMaxK];
  for (int64_t r = 0; r < nS; ++r) {
    uint32_t S = colex_unrank(t, r);
    int m = 0;
    for (int c = 0; c < k; ++c)
      if (S >> c & 1u) elem[m++] = c;
    for (int64_t q = 0; q < nq; ++q) {
      uint32_t pos = colex_unrank(a, q);  // positions within S
      uint32_t S1 = 0;
      for (int i = 0; i < t; ++i)
        if (pos >> i & 1u) S1 |= 1u << elem[i];
      uint32_t S2 = S & ~S1;
      out[(size_t)(q * nS + r)] = (uint32_t)colex_rank(S1) | ((uint32_t)colex_rank(S2) << 16);
    }
  }
  return out;
}

std::vector<uint16_t> drop_table(int k, int t) {
  const int64_t nS = binom(k, t);
  std::vector<uint16_t> out((size_t)(nS * 16), 0xFFFF);
  for (int64_t r = 0; r < nS; ++r) {
    uint32_t S = colex_unrank(t, r);
    for (int c = 0; c < k; ++c)
      if (S >> c & 1u) out[(size_t)(r * 16 + c)] = (uint16_t)colex_rank(S & ~(1u << c));
  }
  return out;
}

// sq_c: drop colour c from the universe (colours above c shift down by one);
// us_c: its inverse (re-insert a gap at c).
uint32_t squeeze(uint32_t mask, int c) { return (mask & ((1u << c) - 1u)) | ((mask >> (c + 1)) << c); }
uint32_t unsqueeze(uint32_t mask, int c) { return (mask & ((1u << c) - 1u)) | ((mask >> c) << (c + 1)); }

int64_t gather_map_ld(int k, int p) { return (binom(k - 1, p - 1) + 7) / 8 * 8; }

std::vector<uint16_t> gather_map(int k, int p, const Layout *lin, const Layout *lout) {
  const int64_t w_in = binom(k - 1, p - 1), ld = gather_map_ld(k, p);
  std::vector<uint16_t> out((size_t)(k * k * ld), 0xFFFF);
  for (int cu = 0; cu < k; ++cu)
    for (int cv = 0; cv < k; ++cv) {
      if (cu == cv) continue;
      for (int64_t q = 0; q < w_in; ++q) {  // storage position q of u's row
        const int64_t r = lin ? lin->rank[(size_t)q] : q;
        const uint32_t Y = unsqueeze(colex_unrank(p - 1, r), cu) | (1u << cu);  // u's colour set
        if (Y >> cv & 1u) continue;                                             // meets v's colour
        const int64_t y = colex_rank(squeeze(Y, cv));
        out[(size_t)((cu * k + cv) * ld + q)] = (uint16_t)(lout ? lout->pos[(size_t)y] : y);
      }
    }
  return out;
}

// Sector-homogeneous storage order of the s-subsets of a K-colour universe
// (build decision R-3): consecutive groups of E sets (E = entries per 32-byte
// sector) that share as many colours as possible, so that a neighbour row's
// sectors whose sets all contain the destination's colour -- never used by
// it -- are as many as possible (they are not read, R-2).  Greedy over
// shared cores of size s-1, s-2, ..., 1 (each core's remaining supersets cut
// into groups of E), the rest in colex order; deterministic.
Layout pack_layout(int K, int s, int E) {
  Layout L;
  const int64_t W = binom(K, s);
  L.rank.resize((size_t)W);
  L.pos.resize((size_t)W);
  std::vector<uint32_t> sets((size_t)W);
  for (int64_t r = 0; r < W; ++r) sets[r] = colex_unrank(s, r);
  std::vector<char> used((size_t)W, 0);
  int64_t n = 0;
  uint64_t rng = 0x9E3779B97F4A7C15ULL;  // fixed-seed xorshift: the order of the cores tried
  auto next = [&]() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
  };
  for (int c = s - 1; c >= 1 && s >= 2; --c) {
    std::vector<uint32_t> cores;
    for (int64_t r = 0; r < binom(K, c); ++r) cores.push_back(colex_unrank(c, r));
    for (size_t i = cores.size(); i > 1; --i) std::swap(cores[i - 1], cores[next() % i]);
    for (bool changed = true; changed;) {
      changed = false;
      for (uint32_t core : cores) {
        std::vector<int64_t> cand;
        for (int64_t r = 0; r < W; ++r)
          if (!used[r] && (sets[r] & core) == core) cand.push_back(r);
        for (size_t i = 0; i + E <= cand.size(); i += E) {
          for (int e = 0; e < E; ++e) {
            used[cand[i + e]] = 1;
            L.rank[(size_t)n++] = (int32_t)cand[i + e];
          }
          changed = true;
        }
      }
    }
  }
  for (int64_t r = 0; r < W; ++r)
    if (!used[r]) L.rank[(size_t)n++] = (int32_t)r;
  for (int64_t q = 0; q < W; ++q) L.pos[(size_t)L.rank[q]] = (int32_t)q;
  return L;
}

Layout identity_layout(int K, int s) {
  Layout L;
  const int64_t W = binom(K, s);
  L.rank.resize((size_t)W);
  std::iota(L.rank.begin(), L.rank.end(), 0);
  L.pos = L.rank;
  return L;
}

std::vector<uint16_t> complement_table(int k, int a) {
  const int64_t nX = binom(k, a);
  const uint32_t full = (k == 32) ? 0xFFFFFFFFu : ((1u << k) - 1u);
  std::vector<uint16_t> out((size_t)nX);
  for (int64_t r = 0; r < nX; ++r) out[(size_t)r] = (uint16_t)colex_rank(full & ~colex_unrank(a, r));
  return out;
}

}  // namespace cc

namespace cc {

// Z-block cover of a combine step (t'; a', p') in the K-colour universe
// (see common.h).  Greedy: take the first uncovered output S in colex
// order, extend it by the colour c that completes the most uncovered
// outputs, and assign every uncovered S_z = Z \ {z} to that block.
std::vector<uint16_t> zblock_table(int K, int ts, int as, int *n_blocks) {
  const int zs = ts + 1, ps = ts - as;
  const int64_t nS = binom(K, ts), na = binom(zs, as), nn = binom(zs, ps);
  const int64_t ld = zblock_ld(ts, as);
  std::vector<char> covered((size_t)nS, 0);
  std::vector<uint16_t> out;
  int nb = 0;
  auto expand = [&](uint32_t Z, uint32_t local) {  // local subset of Z's positions -> global mask
    uint32_t g = 0;
    int pos = 0;
    for (int c = 0; c < K; ++c)
      if (Z >> c & 1u) {
        if (local >> pos & 1u) g |= 1u << c;
        ++pos;
      }
    return g;
  };
  for (int64_t r = 0; r < nS; ++r) {
    if (covered[r]) continue;
    const uint32_t S = colex_unrank(ts, r);
    int best_c = -1, best = -1;
    for (int c = 0; c < K; ++c) {
      if (S >> c & 1u) continue;
      const uint32_t Z = S | 1u << c;
      int gain = 0;
      for (int z = 0; z < K; ++z)
        if (Z >> z & 1u) gain += !covered[colex_rank(Z & ~(1u << z))];
      if (gain > best) {
        best = gain;
        best_c = c;
      }
    }
    const uint32_t Z = S | 1u << best_c;
    const size_t base = out.size();
    out.resize(base + (size_t)ld, 0);
    for (int64_t i = 0; i < na; ++i) out[base + i] = (uint16_t)colex_rank(expand(Z, colex_unrank(as, i)));
    for (int64_t i = 0; i < nn; ++i) out[base + na + i] = (uint16_t)colex_rank(expand(Z, colex_unrank(ps, i)));
    for (int zl = 0; zl < zs; ++zl) {  // output S_z = Z minus its zl-th element (local order)
      const uint32_t Sz = expand(Z, ((1u << zs) - 1) & ~(1u << zl));
      const int64_t rz = colex_rank(Sz);
      out[base + na + nn + zl] = covered[rz] ? 0xFFFF : (uint16_t)rz;
      covered[rz] = 1;
    }
    ++nb;
  }
  *n_blocks = nb;
  return out;
}

int64_t zblock_ld(int ts, int as) {
  const int zs = ts + 1;
  return (binom(zs, as) + binom(zs, ts - as) + zs + 7) / 8 * 8;
}

}  // namespace cc

namespace cc {

std::vector<uint32_t> skip_table(int k, int p, int elem, int *words, const Layout *lin) {
  const int K = k - 1, s = p - 1;
  const int64_t W = binom(K, s);
  const int vw = 16 / elem, se = 32 / elem;  // entries per 16-byte vector / 32-byte sector
  const int64_t nvec = (W + vw - 1) / vw;
  const int nw = (int)((nvec + 31) / 32) + 4;  // + slack: the kernel may address (pass, j) words past the row
  std::vector<uint32_t> out((size_t)K * nw, 0);
  std::vector<uint32_t> sets((size_t)W);
  for (int64_t q = 0; q < W; ++q) sets[q] = colex_unrank(s, lin ? lin->rank[(size_t)q] : q);  // storage order
  for (int c = 0; c < K; ++c)
    for (int64_t vi = 0; vi < nvec; ++vi) {
      const int64_t s0 = vi * vw / se * se;
      bool useless = true;
      for (int64_t e = s0; e < s0 + se && useless; ++e)
        if (e < W && !(sets[e] >> c & 1u)) useless = false;
      if (useless) out[(size_t)c * nw + vi / 32] |= 1u << (vi % 32);
    }
  *words = nw;
  return out;
}

}  // namespace cc
