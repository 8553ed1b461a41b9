// graph.cpp -- CSR validation and the 1D vertex partition (host).
//
// PAPER.md Alg. 2 line 2 (line 209): "G(V,E) is randomly partitioned into P
// processes"; lines 374-382: local neighbours N_l and remote neighbours
// N_{r,w}.  Here: isolated vertices are dropped (their rows are zero for
// templates of >= 2 vertices), a seeded shuffle of the remaining vertices is
// cut into contiguous ranges balanced on (degree + 16), and each rank's
// range is ordered hubs-first (degree descending) so that heavy vertices are
// scheduled first and sit contiguously in memory.  Each rank keeps a local
// CSR whose column ids index [owned rows | halo rows]; halo rows are grouped
// by owning peer, and the peer's send list is the same sorted set.
#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "common.h"

namespace cc {

namespace {
inline uint64_t perm_mix(uint64_t x) {  // relabel shuffle RNG (internal; results never depend on it)
  x ^= x >> 31;
  x *= 0x7FB5D329728EA185ULL;
  x ^= x >> 27;
  x *= 0x81DADEF4BC2DD44DULL;
  x ^= x >> 33;
  return x;
}
}  // namespace

HostGraph validate_graph(int64_t n, const int64_t *row_ptr, const int32_t *col) {
  if (n < 0 || n >= (int64_t)INT32_MAX) throw Error(CC_ERR_GRAPH, "n must be in [0, 2^31 - 1)");
  if (n > 0 && !row_ptr) throw Error(CC_ERR_ARG, "row_ptr is NULL");
  HostGraph g;
  g.n = n;
  if (n == 0) {
    g.rp_own.assign(1, 0);
    g.rp = g.rp_own.data();
    return g;
  }
  g.rp = row_ptr;
  if (g.rp[0] != 0) throw Error(CC_ERR_GRAPH, "row_ptr[0] != 0");
  for (int64_t v = 0; v < n; ++v)
    if (g.rp[v + 1] < g.rp[v]) throw Error(CC_ERR_GRAPH, "row_ptr decreases at row " + std::to_string(v));
  const int64_t nnz = g.rp[n];
  g.nnz = nnz;
  if (nnz > 0 && !col) throw Error(CC_ERR_ARG, "col is NULL");
  // rows sorted already (the usual case): validate the caller's array in place
  int64_t unsorted = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : unsorted)
  for (int64_t v = 0; v < n; ++v) unsorted += !std::is_sorted(col + g.rp[v], col + g.rp[v + 1]);
  if (unsorted) {
    g.col_own.assign(col, col + nnz);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t v = 0; v < n; ++v) std::sort(g.col_own.data() + g.rp[v], g.col_own.data() + g.rp[v + 1]);
    g.col = g.col_own.data();
  } else {
    g.col = col;
  }
  int64_t bad_range = INT64_MAX, bad_loop = INT64_MAX, bad_dup = INT64_MAX, bad_sym = INT64_MAX;
#pragma omp parallel for schedule(dynamic, 4096) reduction(min : bad_range, bad_loop, bad_dup)
  for (int64_t v = 0; v < n; ++v) {
    const int32_t *b = g.col + g.rp[v], *e = g.col + g.rp[v + 1];
    bool range_ok = true;
    for (const int32_t *p = b; p < e; ++p)
      if (*p < 0 || *p >= n) range_ok = false;
    if (!range_ok) { bad_range = std::min<int64_t>(bad_range, v); continue; }
    for (const int32_t *p = b; p < e; ++p) {
      if (*p == v) bad_loop = std::min<int64_t>(bad_loop, v);
      if (p > b && p[-1] == *p) bad_dup = std::min<int64_t>(bad_dup, v);
    }
  }
  if (bad_range != INT64_MAX) throw Error(CC_ERR_GRAPH, "neighbour id out of [0, n) in row " + std::to_string(bad_range));
  if (bad_loop != INT64_MAX) throw Error(CC_ERR_GRAPH, "self-loop at vertex " + std::to_string(bad_loop));
  if (bad_dup != INT64_MAX) throw Error(CC_ERR_GRAPH, "duplicate neighbour in row " + std::to_string(bad_dup));
#pragma omp parallel for schedule(dynamic, 4096) reduction(min : bad_sym)
  for (int64_t v = 0; v < n; ++v) {
    for (int64_t e = g.rp[v]; e < g.rp[v + 1]; ++e) {
      int32_t u = g.col[e];
      if (!std::binary_search(g.col + g.rp[u], g.col + g.rp[u + 1], (int32_t)v)) {
        bad_sym = std::min<int64_t>(bad_sym, v);
        break;
      }
    }
  }
  if (bad_sym != INT64_MAX) throw Error(CC_ERR_GRAPH, "adjacency not symmetric at row " + std::to_string(bad_sym));
  return g;
}

RankPart partition_graph(const HostGraph &g, int world, int rank, uint64_t relabel_seed) {
  if (world < 1 || rank < 0 || rank >= world || world > 64) throw Error(CC_ERR_ARG, "bad world/rank");
  RankPart R;
  R.world = world;
  R.rank = rank;
  R.n_global = g.n;
  const int64_t n = g.n;
  std::vector<int32_t> nz;
  for (int64_t v = 0; v < n; ++v) {
    if (g.rp[v + 1] > g.rp[v]) nz.push_back((int32_t)v);
    else R.iso_orig.push_back((int32_t)v);
  }
  const int64_t nn = (int64_t)nz.size();
  auto deg = [&](int32_t v) { return g.rp[v + 1] - g.rp[v]; };
  if (world > 1) {  // seeded Fisher-Yates
    for (int64_t i = nn - 1; i > 0; --i) {
      uint64_t r = perm_mix(relabel_seed ^ perm_mix((uint64_t)i));
      int64_t j = (int64_t)(r % (uint64_t)(i + 1));
      std::swap(nz[i], nz[j]);
    }
  }
  // contiguous ranges balanced on deg + 16
  std::vector<int64_t> bound(world + 1, nn);
  bound[0] = 0;
  {
    double total = 0;
    for (int32_t v : nz) total += (double)(deg(v) + 16);
    double acc = 0;
    int r = 1;
    for (int64_t i = 0; i < nn && r < world; ++i) {
      while (r < world && acc >= total * r / world) bound[r++] = i;
      acc += (double)(deg(nz[i]) + 16);
    }
    while (r < world) bound[r++] = nn;
  }
  // hubs first within each range; ties by original id (measured: keeping the
  // generator's id order makes the gathers 20% slower on config 3, a BFS
  // (Cuthill-McKee) order from the hubs 27% slower)
  for (int r = 0; r < world; ++r)
    std::sort(nz.begin() + bound[r], nz.begin() + bound[r + 1], [&](int32_t a, int32_t b) {
      int64_t da = deg(a), db = deg(b);
      return da != db ? da > db : a < b;
    });
  std::vector<int32_t> internal(n, -1);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nn; ++i) internal[nz[i]] = (int32_t)i;
  auto owner = [&](int32_t gid) {
    return (int)(std::upper_bound(bound.begin(), bound.end(), (int64_t)gid) - bound.begin()) - 1;
  };
  const int64_t lo = bound[rank], hi = bound[rank + 1];
  R.n_own = hi - lo;
  R.own_orig.assign(nz.begin() + lo, nz.begin() + hi);
  // halo
  std::vector<int32_t> halo;
  if (world > 1) {
    for (int64_t i = lo; i < hi; ++i) {
      int32_t v = nz[i];
      for (int64_t e = g.rp[v]; e < g.rp[v + 1]; ++e) {
        int32_t gid = internal[g.col[e]];
        if (gid < lo || gid >= hi) halo.push_back(gid);
      }
    }
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  }
  R.n_halo = (int64_t)halo.size();
  R.halo_orig.resize(halo.size());
  for (size_t h = 0; h < halo.size(); ++h) R.halo_orig[h] = nz[halo[h]];
  R.recv_off.assign(world + 1, 0);
  for (int q = 0; q <= world; ++q)
    R.recv_off[q] = std::lower_bound(halo.begin(), halo.end(), (int32_t)bound[q]) - halo.begin();
  // local CSR
  R.rp.assign(R.n_own + 1, 0);
  for (int64_t i = 0; i < R.n_own; ++i) R.rp[i + 1] = R.rp[i] + deg(R.own_orig[i]);
  R.col.resize(R.rp[R.n_own]);
  R.mid.resize(R.n_own);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < R.n_own; ++i) {
    int32_t v = R.own_orig[i];
    int32_t *out = R.col.data() + R.rp[i];
    int64_t m = 0;
    for (int64_t e = g.rp[v]; e < g.rp[v + 1]; ++e) {
      int32_t gid = internal[g.col[e]];
      int32_t loc;
      if (gid >= lo && gid < hi) loc = (int32_t)(gid - lo);
      else loc = (int32_t)(R.n_own + (std::lower_bound(halo.begin(), halo.end(), gid) - halo.begin()));
      out[m++] = loc;
    }
    std::sort(out, out + m);
    R.mid[i] = R.rp[i] + (std::lower_bound(out, out + m, (int32_t)R.n_own) - out);
  }
  // send lists: owned rows adjacent to each peer's range, ascending local index
  R.send_off.assign(world + 1, 0);
  if (world > 1) {
    std::vector<std::vector<int32_t>> lists(world);
    for (int64_t i = 0; i < R.n_own; ++i) {
      uint64_t peers = 0;
      for (int64_t e = R.mid[i]; e < R.rp[i + 1]; ++e) {
        int32_t gid = halo[R.col[e] - R.n_own];
        peers |= 1ull << owner(gid);
      }
      for (int q = 0; q < world; ++q)
        if (peers >> q & 1ull) lists[q].push_back((int32_t)i);
    }
    for (int q = 0; q < world; ++q) R.send_off[q + 1] = R.send_off[q] + (int64_t)lists[q].size();
    R.send_idx.reserve(R.send_off[world]);
    for (int q = 0; q < world; ++q) R.send_idx.insert(R.send_idx.end(), lists[q].begin(), lists[q].end());
  }
  return R;
}

std::vector<int64_t> peer_bounds(const RankPart &R) {
  const int W = R.world;
  const int64_t n = R.n_own;
  std::vector<int64_t> b((size_t)(W + 1) * n);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    const int32_t *row = R.col.data();
    for (int q = 0; q <= W; ++q) {
      const int64_t lo = R.mid[i], hi = R.rp[i + 1];
      b[(size_t)q * n + i] =
          q == W ? hi : std::lower_bound(row + lo, row + hi, (int32_t)(R.n_own + R.recv_off[q])) - row;
    }
  }
  return b;
}

ExchangeModel model_exchange(const RankPart &R, const std::vector<int64_t> &b, double w) {
  // Rates (reading): NVLink 5 through NVSwitch, 900 GB/s
  // per direction, ~700 GB/s achieved by one peer-to-peer stream; the
  // neighbour-sum gathers move ~7 TB/s of algorithmic bytes on config 3
  // (profiles/r1); a ring step costs ~20 us of NCCL group launch.
  ExchangeModel m;
  m.link_bps = 700e9;
  m.gather_bps = 7e12;
  const double step_s = 20e-6;
  const int W = R.world, me = R.rank;
  const int64_t n = R.n_own;
  std::vector<double> nnz(W, 0.0), items(W, 0.0);
  double local = 0;
  for (int64_t i = 0; i < n; ++i) {
    local += (double)(R.mid[i] - R.rp[i]);
    for (int q = 0; q < W; ++q) {
      const int64_t d = b[(size_t)(q + 1) * n + i] - b[(size_t)q * n + i];
      nnz[q] += (double)d;
      items[q] += d > 0;
    }
  }
  double items_remote = 0;
  for (int64_t i = 0; i < n; ++i) items_remote += R.rp[i + 1] > R.mid[i];
  auto gather_s = [&](double entries, double touched) {  // index + rows read, N'' rows read and written
    return (entries * (4.0 + w) + touched * 2.0 * w) / m.gather_bps;
  };
  const double t_local = gather_s(local, 0.0);
  double halo = 0, remote = 0;
  for (int q = 0; q < W; ++q) {
    halo += (double)(R.recv_off[q + 1] - R.recv_off[q]) * w / m.link_bps;
    remote += nnz[q];
  }
  m.grouped_s = std::max(halo + step_s, t_local) + gather_s(remote, items_remote);
  double comm = 0, t = t_local;
  for (int r = 1; r < W; ++r) {
    const int src = (me - r + W) % W;
    comm += step_s + (double)(R.recv_off[src + 1] - R.recv_off[src]) * w / m.link_bps;
    t = std::max(t, comm) + gather_s(nnz[src], items[src]);
  }
  m.ring_s = t;
  return m;
}

}  // namespace cc
