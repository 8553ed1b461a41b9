// exec.cu -- graph upload, plan upload and the per-colouring step executor.
//
// One cc_count_colorful = PAPER.md Alg. 1 lines 8-10 (Eq. 2) for one
// colouring, distributed as Alg. 2 (lines 199-243) when world > 1:
//   colour-sort the neighbour ranges (once per colouring);
//   for each step (t; a, p) of the plan (sub-templates in reverse partition
//   order):
//     N'' <- neighbour sum of the passive table (once per distinct passive);
//            world > 1: the passive table's boundary rows are exchanged with
//            grouped NCCL send/recv on a comm stream while the local part of
//            the neighbour sum runs (pipelining);
//     T'  <- split-sum combine of the active table with N'' (a >= 2), or
//            T' = N'' itself (a = 1: no work in the compressed layout);
//   X = sum_v of the root step (fp64), all-reduced over ranks (line 237).
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cmath>
#include <functional>
#include <cstring>

#include "ctx.h"

namespace cc {

namespace {

void build_pass(cc_ctx *c, const std::vector<int64_t> &beg, const std::vector<int64_t> &end, bool skip_empty,
                Pass &w) {
  // segment length s of Alg. 4; colour-group offsets are stored as uint16.
  // Auto: with W adjacency entries per resident warp (16 per SM), s ~
  // 4 sqrt(20 W) rounded to a power of two in [64, 4096], and 4096 once W >=
  // 100K (measured optimum with the row-parallel kernel for long narrow
  // lists: configs[1] 512, [2] 2048-4096, [3] 4096 -- a long hub list on one
  // warp is the tail of small graphs, partial-row traffic the cost of short
  // segments on big ones; with sub-warp rings only it was 128 / 512 / 4096)
  int64_t L = c->opt.segment_len;
  if (L <= 0) {
    int64_t nnz_all = 0;
    for (int64_t v = 0; v < (int64_t)beg.size(); ++v) nnz_all += end[v] - beg[v];
    const double W = (double)nnz_all / (double)(std::max(c->num_sms, 1) * 16);
    L = 4096;
    if (W < 100000.0) {
      L = 64;
      while (L < 4096 && (double)(2 * L) <= std::sqrt(320.0 * W) * 1.414) L *= 2;
    }
  }
  L = std::min<int64_t>(L, 65535);
  w.seg_len = L;
  std::vector<int32_t> light, seg_v, seg_hv, hv_first, hv_nseg;
  std::vector<int64_t> seg_b, seg_e;
  int64_t nnz = 0;
  for (int64_t v = 0; v < (int64_t)beg.size(); ++v) {
    const int64_t d = end[v] - beg[v];
    nnz += d;
    if (d == 0 && skip_empty) continue;
    if (d > L) {
      const int64_t ns = (d + L - 1) / L;
      hv_first.push_back((int32_t)seg_v.size());
      hv_nseg.push_back((int32_t)ns);
      for (int64_t s = 0; s < ns; ++s) {
        seg_v.push_back((int32_t)v);
        seg_hv.push_back((int32_t)(hv_first.size() - 1));
        seg_b.push_back(beg[v] + s * L);
        seg_e.push_back(std::min(end[v], beg[v] + (s + 1) * L));
      }
    } else {
      light.push_back((int32_t)v);
    }
  }
  w.nnz = nnz;
  w.n_light = (int64_t)light.size();
  // adjacency entries before each item (segments first, then light items)
  w.pref.assign((size_t)(seg_v.size() + light.size() + 1), 0);
  for (size_t i = 0; i < seg_v.size(); ++i) w.pref[i + 1] = w.pref[i] + (seg_e[i] - seg_b[i]);
  for (size_t i = 0; i < light.size(); ++i)
    w.pref[seg_v.size() + i + 1] = w.pref[seg_v.size() + i] + (end[light[i]] - beg[light[i]]);
  {  // light items are in internal (degree-descending) order: the <= 8-neighbour tail
    int64_t i = (int64_t)light.size();
    while (i > 0 && end[light[i - 1]] - beg[light[i - 1]] <= 8) --i;
    w.small_from = (int64_t)seg_v.size() + i;
    for (int q = 0; q < 8; ++q) {
      int64_t iq = (int64_t)light.size();
      while (iq > 0 && end[light[iq - 1]] - beg[light[iq - 1]] <= (8 << q)) --iq;
      w.split[q] = (int64_t)seg_v.size() + iq;
    }
  }
  w.n_seg = (int64_t)seg_v.size();
  w.n_hv = (int64_t)hv_first.size();
  w.light_h = light;
  w.max_heavy_v = seg_v.empty() ? -1 : *std::max_element(seg_v.begin(), seg_v.end());
  w.light = c->pupload(light);
  w.seg_v = c->pupload(seg_v);
  w.seg_hv = c->pupload(seg_hv);
  w.hv_first = c->pupload(hv_first);
  w.hv_nseg = c->pupload(hv_nseg);
  w.seg_b = c->pupload(seg_b);
  w.seg_e = c->pupload(seg_e);
  w.goff = c->pmalloc<uint16_t>((size_t)std::max<int64_t>(w.items(), 1) * 16);
  w.desc = c->pmalloc<dev::ItemDesc>((size_t)std::max<int64_t>(w.items(), 1));
  c->max_hv = std::max(c->max_hv, w.n_hv);
  c->max_seg = std::max(c->max_seg, w.n_seg);
}

// Stream-ordered buffers with shared ownership (see Buf).  Whatever is still
// owned when the executor unwinds (an exception: OOM, a NCCL error, a
// rendezvous timeout) is released by the destructor, so a failed count does
// not leave tens of GB in the pool.
struct Bufs {
  cc_ctx *c;
  std::vector<Buf> pool;
  explicit Bufs(cc_ctx *cx) : c(cx) { pool.reserve(256); }
  ~Bufs() {
    for (auto &b : pool)
      if (b.p && b.owned) {
        cudaFreeAsync(b.p, c->s_main);  // no throw from a destructor
        c->cur_bytes -= b.bytes;
        b.p = nullptr;
      }
  }
  Bufs(const Bufs &) = delete;
  Bufs &operator=(const Bufs &) = delete;
  int make(size_t bytes) {
    pool.push_back({c->amalloc(bytes, c->s_main), bytes, 1, true});
    return (int)pool.size() - 1;
  }
  int alias(void *p, size_t bytes) {  // a buffer owned elsewhere (table cache)
    pool.push_back({p, bytes, 1, false});
    return (int)pool.size() - 1;
  }
  void ref(int b) { pool[b].refs++; }
  void unref(int b) {
    if (b < 0) return;
    if (--pool[b].refs == 0 && pool[b].owned) c->afree(pool[b].p, pool[b].bytes, c->s_main);
  }
  void *ptr(int b) const { return b < 0 ? nullptr : pool[b].p; }
};

// A stream-ordered scratch buffer released on scope exit (also when a launch
// or a NCCL call throws).
struct ScopedAsync {
  cc_ctx *c;
  cudaStream_t s;
  size_t bytes = 0;
  void *p = nullptr;
  ScopedAsync(cc_ctx *cx, size_t b, cudaStream_t st) : c(cx), s(st), bytes(b) {
    if (b) p = c->amalloc(b, s);
  }
  ~ScopedAsync() {
    if (p) {
      cudaFreeAsync(p, s);
      c->cur_bytes -= bytes;
    }
  }
  ScopedAsync(const ScopedAsync &) = delete;
  ScopedAsync &operator=(const ScopedAsync &) = delete;
};

}  // namespace

void allreduce_host(cc_ctx *c, std::vector<double> &v);

void load_graph(cc_ctx *c, const HostGraph &g) {
  ++c->epoch;
  c->part = partition_graph(g, c->pworld(), c->pworld() == 1 ? 0 : c->opt.rank, c->opt.relabel_seed);
  const auto &R = c->part;
  c->n_global = g.n;
  {
    int64_t nz = 0;
    for (int64_t v = 0; v < g.n; ++v) nz += g.rp[v + 1] > g.rp[v];
    c->avg_degree = nz ? (double)g.nnz / (double)nz : 0.0;
  }
  c->n_own = R.n_own;
  c->n_halo = R.n_halo;
  c->n_rows = R.n_own + R.n_halo;
  c->d_rp = c->pupload(R.rp);
  c->d_col = c->pupload(R.col);
  c->d_col_sorted = c->pmalloc<int32_t>(std::max<size_t>(R.col.size(), 1));
  std::vector<int32_t> orig(R.own_orig);
  orig.insert(orig.end(), R.halo_orig.begin(), R.halo_orig.end());
  orig.insert(orig.end(), R.iso_orig.begin(), R.iso_orig.end());
  c->n_crow = (int64_t)orig.size();
  c->d_orig = c->pupload(orig);
  c->d_colors = c->pmalloc<uint8_t>((size_t)std::max<int64_t>(c->n_crow, 1));
  c->d_color_stage = c->pmalloc<uint8_t>((size_t)std::max<int64_t>(c->n_global, 1));
  c->d_bad = c->pmalloc<unsigned>(1);
  std::vector<int64_t> beg(R.rp.begin(), R.rp.end() - 1), end(R.rp.begin() + 1, R.rp.end());
  build_pass(c, beg, end, false, c->p_full);
  c->p_full.beg = c->d_rp;
  c->p_full.end = c->d_rp + 1;
  c->p_full.col_sorted = c->d_col_sorted;  // world > 1: its own buffer, allocated for the fused root
  if (c->pworld() > 1) {
    const int W = c->pworld(), me = c->opt.rank;
    c->d_mid = c->pupload(R.mid);
    c->d_send_idx = c->pupload(R.send_idx);
    build_pass(c, beg, R.mid, false, c->p_local);
    c->p_local.beg = c->d_rp;
    c->p_local.end = c->d_mid;
    c->p_local.col_sorted = c->d_col_sorted;
    // exchange schedule (Alg. 3 "Adaptive-Group"): the same on every rank --
    // the cost model's maximum over the ranks when auto
    const std::vector<int64_t> bnd = peer_bounds(R);
    {
      const ExchangeModel m = model_exchange(R, bnd, 1024.0);
      std::vector<double> v(2 * (size_t)W, 0.0);
      v[2 * me] = m.grouped_s;
      v[2 * me + 1] = m.ring_s;
      allreduce_host(c, v);
      c->xmodel[0] = c->xmodel[1] = 0;
      for (int q = 0; q < W; ++q) {
        c->xmodel[0] = std::max(c->xmodel[0], v[2 * q]);
        c->xmodel[1] = std::max(c->xmodel[1], v[2 * q + 1]);
      }
    }
    c->xmode = c->opt.exchange != CC_EXCHANGE_AUTO ? c->opt.exchange
               : c->xmodel[1] < c->xmodel[0]        ? CC_EXCHANGE_RING
                                                    : CC_EXCHANGE_GROUPED;
    if (c->xmode == CC_EXCHANGE_ALLTOALL || c->xmode == CC_EXCHANGE_DEVICE) {
      // every rank's receive offsets (row q of W + 1 entries), from one all-reduce
      std::vector<double> v((size_t)W * (W + 1), 0.0);
      for (int q = 0; q <= W; ++q) v[(size_t)me * (W + 1) + q] = (double)R.recv_off[q];
      allreduce_host(c, v);
      c->max_halo = 0;
      c->a2a_rows = 0;
      std::vector<int64_t> dst_row(W, 0);  // where this rank's rows start in peer q's halo
      for (int p = 0; p < W; ++p) {
        c->max_halo = std::max<int64_t>(c->max_halo, (int64_t)v[(size_t)p * (W + 1) + W]);
        for (int q = 0; q < W; ++q)
          c->a2a_rows = std::max<int64_t>(c->a2a_rows, (int64_t)(v[(size_t)p * (W + 1) + q + 1] - v[(size_t)p * (W + 1) + q]));
      }
      for (int q = 0; q < W; ++q) dst_row[q] = (int64_t)v[(size_t)q * (W + 1) + me];
      if (c->xmode == CC_EXCHANGE_DEVICE) devx_init(c, dst_row);
    }
    if (c->xmode == CC_EXCHANGE_RING) {
      // one remote pass per source peer: its neighbours of each owned row
      const int64_t n = R.n_own;
      int64_t *d_b = c->pupload(bnd);
      c->p_peer.assign(W, Pass());
      for (int q = 0; q < W; ++q) {
        if (q == me || R.recv_off[q + 1] == R.recv_off[q]) continue;
        std::vector<int64_t> b0(bnd.begin() + (size_t)q * n, bnd.begin() + (size_t)(q + 1) * n),
            b1(bnd.begin() + (size_t)(q + 1) * n, bnd.begin() + (size_t)(q + 2) * n);
        Pass &w = c->p_peer[q];
        build_pass(c, b0, b1, true, w);
        w.beg = d_b + (size_t)q * n;
        w.end = d_b + (size_t)(q + 1) * n;
        w.col_sorted = c->d_col_sorted;
      }
    } else {
      build_pass(c, R.mid, end, true, c->p_remote);
      c->p_remote.beg = c->d_mid;
      c->p_remote.end = c->d_rp + 1;
      c->p_remote.col_sorted = c->d_col_sorted;
    }
    c->p_full.col_sorted = nullptr;
    c->d_col_sorted_full = nullptr;
  }
  // device-initiated exchange: halo rows always in (double-buffered) windows
  c->chunked = c->pworld() > 1 && (c->chunk_cols > 0 || c->xmode == CC_EXCHANGE_DEVICE);
  c->d_arrive = c->pmalloc<unsigned int>((size_t)std::max<int64_t>(c->max_hv, 1));
  c->arrive_cap = std::max<int64_t>(c->max_hv, 1);
  c->has_graph = true;
  c->sorted_valid = c->full_sorted_valid = false;
}

void replan(cc_ctx *c, bool fixed) {
  ++c->epoch;
  PlanOpts o;
  o.auto_root = !(fixed || c->opt.fixed_root);
  o.elem = c->elem();
  o.kc = c->user_kc;
  if (c->has_graph && c->avg_degree > 0) o.avg_degree = c->avg_degree;  // rank-invariant (global graph)
  c->plan = make_plan((int)c->user_parent.size(), c->user_parent.data(), &o);
  if (c->has_graph) upload_template(c);
}

void upload_template(cc_ctx *c) {
  ++c->epoch;
  for (auto *p : c->d_split) c->pfree(p);
  for (auto *p : c->d_ztab) c->pfree(p);
  for (auto *p : c->d_map) c->pfree(p);
  for (auto *p : c->d_skip) c->pfree(p);
  c->pfree(c->d_comp);
  c->d_split.assign(c->plan.steps.size(), nullptr);
  c->d_ztab.assign(c->plan.steps.size(), nullptr);
  c->zblocks.assign(c->plan.steps.size(), 0);
  c->d_map.assign(kMaxK + 1, nullptr);
  c->d_skip.assign(kMaxK + 1, nullptr);
  c->skip_words.assign(kMaxK + 1, 0);
  c->d_comp = nullptr;
  const int k = c->plan.colours();
  // storage order of the compressed columns of every table size t (R-3):
  // sector-homogeneous for t >= 3; colex for t <= 2 (the leaf level and its
  // lift are written by the colour sort in colex order)
  c->lay.assign(kMaxK + 2, Layout());
  for (int t = 1; t <= k; ++t)
    c->lay[t] = (t >= 3 && c->knobs.layout > 0)
                    ? pack_layout(k - 1, t - 1, (32 << (c->knobs.layout - 1)) / c->elem())  // groups of 32 B, 64 B, 128 B
                    : identity_layout(k - 1, t - 1);
  const auto &L = c->lay;
  for (size_t s = 0; s < c->plan.steps.size(); ++s) {
    const Step &st = c->plan.steps[s];
    // compressed universe: k-1 colours, sets of size t-1 split into (a-1, p);
    // the root of a template with as many vertices as colours pairs each
    // active set with its complement, otherwise the root is a full combine.
    // Indices are storage positions: actives in L[a], neighbour sums of a
    // passive of size p in L[p + 1], outputs in L[t].
    if (st.out < 0 && c->plan.k == k) {
      if (st.a > 1) {
        std::vector<uint16_t> comp = complement_table(k - 1, st.a - 1);
        std::vector<uint16_t> cp(comp.size());
        for (size_t q = 0; q < comp.size(); ++q) cp[q] = (uint16_t)L[st.p + 1].pos[comp[(size_t)L[st.a].rank[q]]];
        c->d_comp = c->pupload(cp);
      }
    } else if (st.a > 1) {
      // rows of the split table padded to a multiple of 8 outputs (16-byte
      // aligned groups of split entries for the combine kernels)
      const std::vector<uint32_t> tab = split_table(k - 1, st.t - 1, st.a - 1);
      const int64_t WO = binom(k - 1, st.t - 1), WOp = (WO + 7) / 8 * 8, nq = binom(st.t - 1, st.a - 1);
      std::vector<uint32_t> pad((size_t)(nq * WOp), 0);
      for (int64_t q = 0; q < nq; ++q)
        for (int64_t o = 0; o < WO; ++o) {
          const uint32_t e = tab[(size_t)(q * WO + L[st.t].rank[(size_t)o])];
          pad[(size_t)(q * WOp + o)] = (uint32_t)L[st.a].pos[e & 0xFFFF] | ((uint32_t)L[st.p + 1].pos[e >> 16] << 16);
        }
      c->d_split[s] = c->pupload(pad);
      if (dev::combine_z_supported(c->elem(), st.t - 1, st.a - 1)) {  // Z-block cover for the register-blocked combine
        int nb = 0;
        std::vector<uint16_t> zt = zblock_table(k - 1, st.t - 1, st.a - 1, &nb);
        const int64_t zld = zblock_ld(st.t - 1, st.a - 1), na = binom(st.t, st.a - 1), nn = binom(st.t, st.p);
        for (int b = 0; b < nb; ++b) {
          uint16_t *e = zt.data() + (size_t)b * zld;
          for (int64_t i = 0; i < na; ++i) e[i] = (uint16_t)L[st.a].pos[e[i]];
          for (int64_t i = na; i < na + nn; ++i) e[i] = (uint16_t)L[st.p + 1].pos[e[i]];
          for (int64_t i = na + nn; i < na + nn + st.t; ++i)
            if (e[i] != 0xFFFF) e[i] = (uint16_t)L[st.t].pos[e[i]];
        }
        c->d_ztab[s] = c->pupload(zt);
        c->zblocks[s] = nb;
      }
    }
    if (st.p > 1 && !c->d_map[st.p]) {
      c->d_map[st.p] = c->pupload(gather_map(k, st.p, &L[st.p], &L[st.p + 1]));
      int nw = 0;
      const std::vector<uint32_t> sk = skip_table(k, st.p, c->elem(), &nw, &L[st.p]);
      c->d_skip[st.p] = c->pupload(sk);
      c->skip_words[st.p] = nw;
    }
  }
}

void launch_colouring(cc_ctx *c, uint64_t seed) {
  if (!c->ev_color[0]) {
    CUDA_OK(cudaEventCreate(&c->ev_color[0]));
    CUDA_OK(cudaEventCreate(&c->ev_color[1]));
  }
  CUDA_OK(cudaEventRecord(c->ev_color[0], c->s_main));
  dev::launch_color(c->d_orig, c->n_crow, seed, c->plan.colours(), c->d_colors, c->s_main);
  c->check_launch();
  CUDA_OK(cudaEventRecord(c->ev_color[1], c->s_main));
  c->has_colors = true;
  c->sorted_valid = c->full_sorted_valid = false;
}

namespace {

void csort(cc_ctx *c, Pass &p) {
  c->stats[3] += dev::launch_csort(p.beg, p.end, c->d_col, c->d_colors, p.view(), p.col_sorted, p.goff,
                                   p.desc, c->num_sms, c->s_main);
  c->check_launch();
  c->stats[1] += (double)p.nnz * 14.0 + (double)p.items() * 64.0;
}

// Fused root: the root step's neighbour sum is consumed in the gather's
// epilogue (X_v into per_vertex) instead of being written to HBM.
struct RootFuse {
  int mode = 0;  // 1: A' = table A; 2: A' = the neighbour sum itself
  const void *A = nullptr;
  int64_t ldA = 0;
  int WA = 0;
  double *per_vertex = nullptr;
};

// The passive rows one neighbour-sum launch reads: columns [c0, c0 + w) of a
// table whose row r starts at base + r * ld elements, P = base + c0 (a halo
// buffer of one column chunk: P is its virtual base -- row n_own is the first
// halo row -- and holds columns c0.. from its column 0).
struct Src {
  const void *P;
  int64_t ld;
  int c0, w;
};

Src table_src(const void *base, int64_t ld, int c0, int w, int elem) {
  return {static_cast<const char *>(base) + (size_t)c0 * elem, ld, c0, w};
}

// N'' (+)= neighbour sum of the passive columns `src` (size p >= 2) over the
// items [from, to) of one pass (to < 0: all).  N is the base of the N'' rows
// (row v at N + v * ldN; a row batch passes a virtual base).  sms: the SMs
// the launch may fill (c->gather_sms).
// A sibling passive summed in the same traversal (one rank, narrow rows):
// its whole table, size p, and its N'' base.
struct PairSrc {
  Src src;
  int p;
  void *N;
};

void gather_pass(cc_ctx *c, Pass &w, const Src &src, int p, void *N, int accumulate, const RootFuse *rf, int sms,
                 int64_t from = 0, int64_t to = -1, const PairSrc *pr = nullptr) {
  const int k = c->plan.colours(), elem = c->elem();
  const int W_out1 = (int)binom(k - 1, p);
  const int W_out = W_out1 + (pr ? (int)binom(k - 1, pr->p) : 0);
  if (to < 0) to = w.items();
  if (from >= to) return;
  dev::GatherArgs a;
  a.beg = w.beg;
  a.end = w.end;
  a.col = w.col_sorted;
  a.goff = w.goff;
  a.desc = w.desc;
  a.colors = c->d_colors;
  a.src = src.P;
  a.ld_src = src.ld;
  a.W_in = src.w;
  a.col_base = src.c0;
  a.item_from = from;
  a.item_to = to;
  {
    // narrow rows: items with more than T neighbours (heavy segments first,
    // then light items in degree order) go to the warp-per-item row-parallel
    // kernel, the rest to the sub-warp rings; T = 8 << q = max(32, s / 16)
    // (measured, profiles/r1/SUMMARY.md); none when segments are <= T long
    int q = 2;  // auto: T = max(32, s / 16)
    while (q < 7 && (8 << (q + 1)) <= w.seg_len / 16) ++q;
    if (c->knobs.narrow_split >= 0) q = std::min(7, c->knobs.narrow_split);
    a.item_split = w.seg_len > (8 << q) ? w.split[q] : 0;
    if (c->knobs.lean_split >= 0) a.lean_split = w.split[std::min(7, c->knobs.lean_split)];
    // first light item of the short tail (k_gather_short takes <= 32 neighbours: one id per lane)
    a.short_from = w.split[std::min(c->knobs.short_lists == 1 ? 2 : 7, std::max(0, c->knobs.short_split))];
  }
  a.map = c->d_map[p];
  a.map_ld = gather_map_ld(k, p);
  if (c->knobs.sector_skip) {
    a.skip = c->d_skip[p];
    a.skip_words = c->skip_words[p];
  }
  // hub rows kept in L2: a fraction of the L2 (rows are degree-ordered, hubs first)
  a.hub_rows = (int64_t)(c->knobs.hub_l2_pct / 100.0 * (double)c->l2_bytes / (double)(a.ld_src * elem));
  a.dst = N;
  a.ld_dst = c->ld_of(W_out1);
  a.W_out = W_out;
  a.k = k;
  if (pr) {  // the virtual row: part 1's whole 16-byte vectors, then part 2
    const int vw = 16 / elem;
    a.nvec1 = (src.w + vw - 1) / vw;
    a.W_in = a.nvec1 * vw + pr->src.w;
    a.src2 = pr->src.P;
    a.ld_src2 = pr->src.ld;
    a.W_in2 = pr->src.w;
    a.map2 = c->d_map[pr->p];
    a.map_ld2 = gather_map_ld(k, pr->p);
    if (c->knobs.sector_skip) {
      a.skip2 = c->d_skip[pr->p];
      a.skip_words2 = c->skip_words[pr->p];
    }
    a.dst2 = pr->N;
    a.ld_dst2 = c->ld_of(W_out - W_out1);
    a.o2 = W_out1;
  }
  a.accumulate = accumulate;
  a.work = w.view();
  a.ld_scratch = W_out;
  const bool segs = from < w.n_seg;
  ScopedAsync scratch(c, segs ? (size_t)w.n_seg * W_out * sizeof(double) : 0, c->s_main);
  if (segs) CUDA_OK(cudaMemsetAsync(c->d_arrive, 0, (size_t)w.n_hv * sizeof(unsigned int), c->s_main));
  a.scratch = static_cast<double *>(scratch.p);
  a.arrive = c->d_arrive;
  if (rf) {
    a.root_mode = rf->mode;
    a.rA = rf->A;
    a.ldA = rf->ldA;
    a.WA = rf->WA;
    a.comp = c->d_comp;
    a.per_vertex = rf->per_vertex;
  }
  // knob nvtx_mark = i > 0: the i-th neighbour-sum pass of the count runs
  // inside the NVTX range "cc_dominant" (bench.py's one-launch ncu pass
  // measures that launch's DRAM traffic with --nvtx-include cc_dominant/)
  const bool mark = c->knobs.nvtx_mark > 0 && ++c->gather_ordinal == c->knobs.nvtx_mark;
  if (mark) nvtxRangePushA("cc_dominant");
  cudaEvent_t b = c->begin(c->s_main);
  c->stats[3] += dev::launch_gather(elem, a, c->knobs, sms, c->s_main);
  c->check_launch();
  c->end(PH_GATHER, c->s_main, b);
  if (mark) nvtxRangePop();
  // algorithmic bytes: index stream + compressed rows of the neighbours whose
  // colour differs from the row vertex's (expected fraction (k-1)/k) + N'' rows
  // written (+ read when accumulating)
  const double nnz = (double)(w.pref[(size_t)to] - w.pref[(size_t)from]);
  const double rows_out = (double)(to - from) - (segs ? (double)(std::min(to, w.n_seg) - from) : 0.0) +
                          (segs ? (double)w.n_hv : 0.0);
  const double rows = nnz * (double)(k - 1) / k * (src.w + (pr ? pr->src.w : 0)) * elem;
  const double out_bytes = rf ? rows_out * (8.0 + (rf->mode == 1 ? (double)rf->WA * elem : 0.0))
                              : rows_out * W_out * elem * (1 + accumulate);
  const double bytes = nnz * 4.0 + rows + out_bytes;
  if (!c->ev_log.empty()) c->gather_log.push_back({c->ev_log.size() - 1, bytes});
  c->stats[0] += nnz * (double)src.w / (double)binom(k - 1, p - 1) * (double)binom(k, p);  // U
  if (pr) c->stats[0] += nnz * (double)binom(k, pr->p);
  c->stats[1] += bytes;
  c->stats[2] += bytes;
}

// Loopback transport (cc_options.loopback): the halo rows of this rank come
// from the peers' send buffers by device copies ordered by the peers' pack
// events; this rank's send buffer is released only after every peer's copy.
void loopback_exchange(cc_ctx *c, void *sendbuf, void *H, int64_t ldH, int elem,
                       std::vector<std::pair<int, cudaEvent_t>> *steps) {
  LoopbackGroup &G = *c->loop;
  const auto &R = c->part;
  const int me = c->opt.rank, W = G.world;
  const bool ring = c->xmode == CC_EXCHANGE_RING;
  cudaEvent_t packed = c->ev(), copied = c->ev();
  CUDA_OK(cudaEventRecord(packed, c->s_comm));
  G.ptr[me] = sendbuf;
  G.offs[me] = R.send_off.data();
  G.ev[me] = packed;
  G.rendezvous();
  for (int r = 1; r < W; ++r) {
    const int q = ring ? (me - r + W) % W : (me + r) % W;  // ring: step r receives from rank - r
    const int64_t nr = R.recv_off[q + 1] - R.recv_off[q];
    if (nr) {
      CUDA_OK(cudaStreamWaitEvent(c->s_comm, G.ev[q], 0));
      CUDA_OK(cudaMemcpyAsync(static_cast<char *>(H) + (size_t)R.recv_off[q] * ldH * elem,
                              static_cast<const char *>(G.ptr[q]) + (size_t)G.offs[q][me] * ldH * elem,
                              (size_t)nr * ldH * elem, cudaMemcpyDeviceToDevice, c->s_comm));
    }
    if (ring && steps) {
      cudaEvent_t e = c->ev();
      CUDA_OK(cudaEventRecord(e, c->s_comm));
      steps->push_back({q, e});
    }
  }
  CUDA_OK(cudaEventRecord(copied, c->s_comm));
  G.ev2[me] = copied;
  G.rendezvous();
  for (int q = 0; q < G.world; ++q)
    if (q != me) CUDA_OK(cudaStreamWaitEvent(c->s_comm, G.ev2[q], 0));
  G.rendezvous();  // every rank has read the slots before they are reused
}

void loopback_allreduce(cc_ctx *c, double *d, size_t count, cudaStream_t s) {
  LoopbackGroup &G = *c->loop;
  const int me = c->opt.rank;
  std::vector<double> h(count);
  CUDA_OK(cudaMemcpyAsync(h.data(), d, count * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  G.vec[me] = h;
  G.rendezvous();
  std::vector<double> sum(count, 0.0);
  for (int r = 0; r < G.world; ++r)  // rank order: the same sum on every rank
    for (size_t i = 0; i < count; ++i) sum[i] += G.vec[r][i];
  G.rendezvous();
  CUDA_OK(cudaMemcpyAsync(d, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaStreamSynchronize(s));
}

// world > 1, on the comm stream (the caller orders it after the producer of
// P): send columns [c0, c0 + w) of this rank's boundary rows of P (owned
// rows, stride ldP) to the peers that need them and receive the peers' rows
// into H (halo row i at H + i * ldH).  Returns an event recorded when every
// halo row has arrived; ring schedule: *steps (nullable) receives (source
// peer, event recorded when that peer's rows have arrived) in step order.
cudaEvent_t exchange_halo(cc_ctx *c, const void *P, int64_t ldP, int64_t c0, int64_t w, void *H, int64_t ldH,
                          std::vector<std::pair<int, cudaEvent_t>> *steps = nullptr) {
  auto &api = nccl();
  const int elem = c->elem();
  const auto &R = c->part;
  const int64_t send_rows = R.send_off[c->pworld()];
  ScopedAsync sb(c, (size_t)send_rows * ldH * elem, c->s_comm);  // released after the sends (stream order)
  void *sendbuf = sb.p;
  cudaEvent_t xb = c->begin(c->s_comm);
  c->stats[3] += dev::launch_pack(elem, P, ldP, c0, w, c->d_send_idx, send_rows, sendbuf, ldH, c->s_comm);
  c->check_launch();
  const ncclDataType_t dt = elem == 8 ? ncclFloat64 : ncclFloat32;
  if (c->loop) {
    loopback_exchange(c, sendbuf, H, ldH, elem, steps);
  } else if (c->xmode == CC_EXCHANGE_ALLTOALL) {
    // ncclAlltoAll needs equal counts: per-peer blocks padded to the largest
    // send count of any rank pair, then each block's rows moved into place
    const int W = c->pworld();
    if (!api.AlltoAll) throw Error(CC_ERR_NCCL, "this NCCL has no ncclAlltoAll");
    const size_t blk = (size_t)c->a2a_rows * ldH * elem;
    ScopedAsync sp(c, blk * W, c->s_comm), rp(c, blk * W, c->s_comm);
    for (int q = 0; q < W; ++q) {
      const int64_t ns = R.send_off[q + 1] - R.send_off[q];
      if (q != c->opt.rank && ns)
        CUDA_OK(cudaMemcpyAsync(static_cast<char *>(sp.p) + blk * q,
                                static_cast<char *>(sendbuf) + (size_t)R.send_off[q] * ldH * elem,
                                (size_t)ns * ldH * elem, cudaMemcpyDeviceToDevice, c->s_comm));
    }
    if (blk) NCCL_OK(api.AlltoAll(sp.p, rp.p, (size_t)c->a2a_rows * ldH, dt, c->comm, c->s_comm));
    for (int q = 0; q < W; ++q) {
      const int64_t nr = R.recv_off[q + 1] - R.recv_off[q];
      if (q != c->opt.rank && nr)
        CUDA_OK(cudaMemcpyAsync(static_cast<char *>(H) + (size_t)R.recv_off[q] * ldH * elem,
                                static_cast<char *>(rp.p) + blk * q, (size_t)nr * ldH * elem,
                                cudaMemcpyDeviceToDevice, c->s_comm));
    }
  } else if (c->xmode == CC_EXCHANGE_RING) {
    // Alg. 3 lines 2-6: step r sends to rank + r and receives from rank - r
    const int W = c->pworld(), me = c->opt.rank;
    for (int r = 1; r < W; ++r) {
      const int dst = (me + r) % W, src = (me - r + W) % W;
      const int64_t ns = R.send_off[dst + 1] - R.send_off[dst];
      const int64_t nr = R.recv_off[src + 1] - R.recv_off[src];
      NCCL_OK(api.GroupStart());
      if (ns)
        NCCL_OK(api.Send(static_cast<char *>(sendbuf) + (size_t)R.send_off[dst] * ldH * elem, (size_t)(ns * ldH), dt,
                         dst, c->comm, c->s_comm));
      if (nr)
        NCCL_OK(api.Recv(static_cast<char *>(H) + (size_t)R.recv_off[src] * ldH * elem, (size_t)(nr * ldH), dt, src,
                         c->comm, c->s_comm));
      NCCL_OK(api.GroupEnd());
      if (steps) {
        cudaEvent_t e = c->ev();
        CUDA_OK(cudaEventRecord(e, c->s_comm));
        steps->push_back({src, e});
      }
    }
  } else {
    NCCL_OK(api.GroupStart());
    for (int q = 0; q < c->pworld(); ++q) {
      if (q == c->opt.rank) continue;
      const int64_t ns = R.send_off[q + 1] - R.send_off[q];
      const int64_t nr = R.recv_off[q + 1] - R.recv_off[q];
      if (ns)
        NCCL_OK(api.Send(static_cast<char *>(sendbuf) + (size_t)R.send_off[q] * ldH * elem, (size_t)(ns * ldH), dt, q,
                         c->comm, c->s_comm));
      if (nr)
        NCCL_OK(api.Recv(static_cast<char *>(H) + (size_t)R.recv_off[q] * ldH * elem, (size_t)(nr * ldH), dt, q,
                         c->comm, c->s_comm));
    }
    NCCL_OK(api.GroupEnd());
  }
  c->end(PH_EXCHANGE, c->s_comm, xb);
  cudaEvent_t recvd = c->ev();
  CUDA_OK(cudaEventRecord(recvd, c->s_comm));
  c->stats[1] += (double)send_rows * w * elem * 2;
  c->stats[9] += (double)(R.recv_off[c->pworld()]) * w * elem;  // halo bytes received
  return recvd;
}

// The comm stream waits for everything queued on the main stream so far.
void comm_after_main(cc_ctx *c) {
  cudaEvent_t e = c->ev();
  CUDA_OK(cudaEventRecord(e, c->s_main));
  CUDA_OK(cudaStreamWaitEvent(c->s_comm, e, 0));
}

// Column chunks of a passive table of W_in columns: widths that
// are multiples of 8 columns (32-byte sectors of fp32 rows), chunk_cols wide.
std::vector<std::pair<int, int>> column_chunks(int W_in, int64_t chunk_cols) {
  std::vector<std::pair<int, int>> out;
  const int w = chunk_cols > 0 ? (int)std::min<int64_t>(W_in, (chunk_cols + 7) / 8 * 8) : W_in;
  for (int c0 = 0; c0 < W_in; c0 += w) out.push_back({c0, std::min(w, W_in - c0)});
  return out;
}

// N'' = neighbour sum of the passive table P (rows of stride ldP, size p >= 2).
// One rank: one launch per column chunk, the later ones accumulating.  The
// 1D partition: the boundary rows of P are exchanged on the comm stream while
// the local part runs; then the remote part --
// grouped: one pass once every halo row is in; ring: one pass per step, each
// as soon as its peer's rows have arrived.  Unchunked, halo rows land in P
// after the owned rows; chunked (c->chunked), per column chunk into one of
// two halo buffers (chunk i + 1 transfers while chunk i is summed): the
// pipeline's memory bound PeakMem^pip.
void aggregate(cc_ctx *c, void *P, int64_t ldP, int p, void *N) {
  const int k = c->plan.colours(), elem = c->elem();
  const int W_in = (int)binom(k - 1, p - 1);
  const auto chunks = column_chunks(W_in, c->chunk_cols);
  if (chunks.size() > 1) c->stats[11] += (double)chunks.size();
  if (c->pworld() == 1) {
    for (size_t i = 0; i < chunks.size(); ++i)
      gather_pass(c, c->p_full, table_src(P, ldP, chunks[i].first, chunks[i].second, elem), p, N, i > 0, nullptr,
                  c->num_sms);
    return;
  }
  const bool ring = c->xmode == CC_EXCHANGE_RING;
  auto remote = [&](const std::vector<std::pair<int, cudaEvent_t>> &steps, const Src &src) {
    for (const auto &st : steps) {
      Pass &w = st.first < 0 ? c->p_remote : c->p_peer[st.first];
      if (!w.items()) continue;
      cudaEvent_t wb = c->begin(c->s_main);  // exposed exchange: s_main idles until the rows are in
      CUDA_OK(cudaStreamWaitEvent(c->s_main, st.second, 0));
      c->end(PH_EXPOSED, c->s_main, wb);
      gather_pass(c, w, src, p, N, 1, nullptr, c->gather_sms(ring));  // ring: the next step transfers meanwhile
    }
  };
  if (!c->chunked) {
    comm_after_main(c);
    std::vector<std::pair<int, cudaEvent_t>> steps;
    cudaEvent_t recvd = exchange_halo(c, P, ldP, 0, ldP, static_cast<char *>(P) + (size_t)c->n_own * ldP * elem, ldP,
                                      ring ? &steps : nullptr);
    gather_pass(c, c->p_local, table_src(P, ldP, 0, W_in, elem), p, N, 0, nullptr, c->gather_sms(true));
    if (!ring) steps.push_back({-1, recvd});
    remote(steps, table_src(P, ldP, 0, W_in, elem));
    CUDA_OK(cudaStreamWaitEvent(c->s_main, recvd, 0));  // the send buffer's release is ordered after every step
    return;
  }
  // chunked: double-buffered halo buffers of the chunk width (device-initiated
  // exchange: the two halves of the registered window)
  const int64_t ldH = c->ld_of(chunks[0].second);
  const bool devx = c->xmode == CC_EXCHANGE_DEVICE;
  const size_t hbytes = (size_t)std::max<int64_t>(devx ? c->max_halo : c->n_halo, 1) * ldH * elem;
  ScopedAsync H0(c, devx ? 0 : hbytes, c->s_main), H1(c, !devx && chunks.size() > 1 ? hbytes : 0, c->s_main);
  void *H[2] = {H0.p, H1.p ? H1.p : H0.p};
  size_t hoff[2] = {0, 0};
  if (devx) {
    char *w = static_cast<char *>(devx_window(c, 2 * hbytes));
    H[0] = w;
    H[1] = w + hbytes;
    hoff[1] = hbytes;
  }
  cudaEvent_t hfree[2] = {nullptr, nullptr};
  comm_after_main(c);  // P produced and the halo buffers allocated
  cudaEvent_t recvd = nullptr;
  for (size_t i = 0; i < chunks.size(); ++i) {
    const int c0 = chunks[i].first, w = chunks[i].second;
    if (hfree[i % 2]) CUDA_OK(cudaStreamWaitEvent(c->s_comm, hfree[i % 2], 0));  // chunk i - 2 summed
    std::vector<std::pair<int, cudaEvent_t>> steps;
    if (devx) {  // the pack kernel stores into the peers' windows (LSA barriers inside)
      cudaEvent_t xb = c->begin(c->s_comm);
      devx_put(c, P, ldP, c0, w, hoff[i % 2], ldH);
      c->end(PH_EXCHANGE, c->s_comm, xb);
      recvd = c->ev();
      CUDA_OK(cudaEventRecord(recvd, c->s_comm));
      c->stats[1] += (double)c->part.send_off[c->pworld()] * w * elem * 2;
      c->stats[9] += (double)c->part.recv_off[c->pworld()] * w * elem;
    } else {
      recvd = exchange_halo(c, P, ldP, c0, w, H[i % 2], ldH, ring ? &steps : nullptr);
    }
    gather_pass(c, c->p_local, table_src(P, ldP, c0, w, elem), p, N, i > 0, nullptr, c->gather_sms(true));
    if (!ring) steps.push_back({-1, recvd});
    // the remote rows of this chunk: halo row j at H + j * ldH, i.e. table row n_own + j
    remote(steps, Src{static_cast<char *>(H[i % 2]) - (size_t)c->n_own * ldH * elem, ldH, c0, w});
    hfree[i % 2] = c->ev();
    CUDA_OK(cudaEventRecord(hfree[i % 2], c->s_main));
  }
  CUDA_OK(cudaStreamWaitEvent(c->s_main, recvd, 0));  // every send buffer released before the halo buffers
}

}  // namespace

// Sum of a small host vector over the ranks (setup only, e.g. the exchange
// model at load time): NCCL all-reduce, or the loopback group's host sum.
void allreduce_host(cc_ctx *c, std::vector<double> &v) {
  void *buf = c->amalloc(v.size() * sizeof(double), c->s_main);
  double *d = static_cast<double *>(buf);
  CUDA_OK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, c->s_main));
  if (c->loop) loopback_allreduce(c, d, v.size(), c->s_main);
  else NCCL_OK(nccl().AllReduce(d, d, v.size(), ncclFloat64, ncclSum, c->comm, c->s_main));
  CUDA_OK(cudaMemcpyAsync(v.data(), d, v.size() * sizeof(double), cudaMemcpyDeviceToHost, c->s_main));
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  c->afree(buf, v.size() * sizeof(double), c->s_main);
}

void LoopbackGroup::rendezvous() {
  std::unique_lock<std::mutex> lk(mu);
  const int64_t gen = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
    return;
  }
  if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return generation != gen; }))
    throw Error(CC_ERR_NCCL, "loopback rendezvous timed out (a rank failed or diverged)");
}

void free_cache(cc_ctx *c, TableCache &cache) {
  for (auto &t : cache.tables) c->afree(t.second.first, t.second.second, c->s_main);
  cache.tables.clear();
  if (cache.hist) c->afree(cache.hist, cache.hist_bytes, c->s_main);
  cache.hist = nullptr;
  cache.sorted = false;
  cache.bytes = 0;
}

namespace {

// The memory plan of one count.  tail >= 0: steps [tail, end)
// run in nb row batches; rc >= 0: step rc (the producer of step tail's
// passive table) is not run in full but per batch, in column chunks of rc_w.
struct MemPlan {
  int tail = -1, nb = 1, rc = -1, rc_w = 0;
};

// Modelled peak of the stream-ordered table memory of run_count's schedule
// (same buffers, same reference counts, same releases), for a memory plan.
double model_peak(cc_ctx *c, const Plan &pl, int64_t rows, int fuse, int defer_lift, int fuse_cr, int last_hist_use,
                  bool per_vertex, const MemPlan &mp) {
  const int k = pl.colours(), elem = c->elem(), nt = (int)pl.tables.size(), sr = (int)pl.steps.size() - 1;
  const int64_t n = c->n_own;
  std::vector<int> last_use(pl.table_last_use), n_last(pl.n_last_use);
  if (mp.tail >= 0) {
    fuse = 0;
    defer_lift = -1;
  } else if (fuse == 2) {
    last_use[pl.steps[sr].passive] = sr;
  }
  if (mp.rc >= 0) {
    const Step &q = pl.steps[mp.rc];
    if (q.active >= 0) last_use[q.active] = sr + 1;
    if (q.p == 1) last_hist_use = sr + 1;
    else n_last[q.passive] = sr + 1;
  }
  auto tbytes = [&](int size) { return (double)rows * c->ld_of(binom(k - 1, size - 1)) * elem; };
  auto nbytes = [&](int p) { return (double)rows * c->ld_of(binom(k - 1, p)) * elem; };
  std::vector<double> bb;  // buffers: bytes (0 = freed)
  std::vector<int> refs;
  double live = 0, peak = 0;
  auto make = [&](double b) {
    bb.push_back(b);
    refs.push_back(1);
    live += b;
    return (int)bb.size() - 1;
  };
  auto unref = [&](int b) {
    if (b >= 0 && --refs[b] == 0) live -= bb[b];
  };
  if (per_vertex || fuse || fuse_cr >= 0 || mp.tail >= 0) make((double)n * 8);
  const double scratch = (double)c->p_full.n_seg * 8;  // x W_out: heavy partial rows of one gather
  std::vector<int> T(nt, -1), Nb(nt, -1);
  int hist = -1;
  const int stop = mp.tail >= 0 ? mp.tail : sr + 1;
  for (int s = 0; s < stop; ++s) {
    const Step &st = pl.steps[s];
    if (s == mp.rc || s == defer_lift) continue;
    double transient = 0;
    if (s == sr && fuse) {
      peak = std::max(peak, live + scratch * binom(k - 1, st.p));
      break;
    }
    int nbuf;
    if (st.p == 1) {
      if (hist < 0) hist = make((double)rows * c->ld_of(k - 1) * elem);
      nbuf = hist;
    } else {
      if (Nb[st.passive] < 0) {
        Nb[st.passive] = make(nbytes(st.p));
        transient = scratch * binom(k - 1, st.p);
      }
      nbuf = Nb[st.passive];
    }
    if (st.out < 0) {
      if (pl.k < k && st.a > 1) transient += tbytes(st.t);
    } else if (st.a == 1) {
      T[st.out] = nbuf;
      ++refs[nbuf];
    } else if (s != fuse_cr) {
      T[st.out] = make(tbytes(st.t));
    }
    peak = std::max(peak, live + transient);
    for (int id = 0; id < nt; ++id) {
      if (T[id] >= 0 && last_use[id] == s) unref(T[id]), T[id] = -1;
      if (Nb[id] >= 0 && n_last[id] == s) unref(Nb[id]), Nb[id] = -1;
    }
    if (hist >= 0 && s == last_hist_use) unref(hist), hist = -2;
  }
  if (mp.tail >= 0) {  // one batch of the tail on top of what is alive
    const int64_t br = (n + mp.nb - 1) / mp.nb + std::max<int64_t>(c->p_full.max_heavy_v + 1 - n / mp.nb, 0);
    const Step &gs = pl.steps[mp.tail];
    double batch = (double)br * c->ld_of(binom(k - 1, gs.p)) * elem + scratch * binom(k - 1, gs.p);
    for (int s = mp.tail; s <= sr; ++s) {
      const Step &st = pl.steps[s];
      if ((st.out >= 0 && st.a > 1 && s != fuse_cr) || (st.out < 0 && pl.k < k && st.a > 1))
        batch += (double)br * c->ld_of(binom(k - 1, st.t - 1)) * elem;
    }
    if (mp.rc >= 0) batch += (double)rows * c->ld_of(mp.rc_w) * elem;
    peak = std::max(peak, live + batch);
  }
  return peak;
}

MemPlan plan_memory(cc_ctx *c, const Plan &pl, int64_t rows, int fuse, int defer_lift, int fuse_cr, int last_hist_use,
                    bool per_vertex) {
  MemPlan none;
  const int sr = (int)pl.steps.size() - 1, forced_nb = c->knobs.tail_batches, forced_w = c->knobs.tail_recompute_cols;
  if (c->pworld() > 1) return none;  // one rank only (the 1D partition bounds memory with chunked halo buffers)
  // plans far below the device's memory need no query (cudaMemGetInfo costs
  // milliseconds of host time, which launch-bound small graphs would see)
  if (forced_nb <= 0 && forced_w <= 0 &&
      model_peak(c, pl, rows, fuse, defer_lift, fuse_cr, last_hist_use, per_vertex, none) < 0.4 * c->total_mem)
    return none;
  // the budget: free device memory + what the stream-ordered pool holds unused, less a margin
  size_t free_b = 0, total_b = 0;
  CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
  cudaMemPool_t pool;
  CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, c->opt.device));
  uint64_t reserved = 0, used = 0;
  CUDA_OK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  CUDA_OK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  const double budget = ((double)free_b + (double)(reserved - std::min(reserved, used))) * 0.97 - 1.5e9;
  if (forced_nb <= 0 && forced_w <= 0 &&
      model_peak(c, pl, rows, fuse, defer_lift, fuse_cr, last_hist_use, per_vertex, none) <= budget)
    return none;
  // the tail: the last step that starts a neighbour sum; every later step must be row-local
  int g = -1;
  for (int s = 0; s <= sr; ++s)
    if (pl.steps[s].p >= 2 && pl.n_first_use[pl.steps[s].passive] == s) g = s;
  if (g < 0) return none;
  for (int s = g + 1; s <= sr; ++s)
    if (pl.steps[s].p >= 2 && pl.n_first_use[pl.steps[s].passive] > g) return none;
  // the producer of the tail's passive table may be recomputed when it is a
  // combine and that table feeds nothing but this neighbour sum
  const int P = pl.steps[g].passive;
  int q = -1;
  for (int s = 0; s < g; ++s)
    if (pl.steps[s].out == P) q = s;
  bool rc_ok = q >= 0 && pl.steps[q].a >= 2 && pl.table_last_use[P] == g;
  for (int s = 0; s <= sr; ++s) rc_ok = rc_ok && pl.steps[s].active != P;
  const int Win = (int)binom(pl.colours() - 1, pl.steps[g].p - 1);
  auto fits = [&](const MemPlan &m) {
    return model_peak(c, pl, rows, fuse, defer_lift, fuse_cr, last_hist_use, per_vertex, m) <= budget;
  };
  if (forced_nb > 0 || forced_w > 0) {  // knobs (tests): this batching, whatever the memory
    MemPlan m;
    m.tail = g;
    m.nb = std::max(1, forced_nb);
    if (forced_w > 0 && rc_ok) {
      m.rc = q;
      m.rc_w = (int)std::min<int64_t>(Win, (forced_w + 7) / 8 * 8);
    }
    return m;
  }
  static const int nbs[] = {2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64};
  for (int nb : nbs) {
    MemPlan m;
    m.tail = g;
    m.nb = nb;
    if (fits(m)) return m;
  }
  if (rc_ok)
    for (int nb : nbs)
      for (int w = (Win + 7) / 8 * 8; w >= 64; w = (w / 2 + 7) / 8 * 8) {
        MemPlan m;
        m.tail = g;
        m.nb = nb;
        m.rc = q;
        m.rc_w = std::min(w, Win);
        if (fits(m)) return m;
        if (w == 64) break;
      }
  return none;  // nothing fits: run as planned (the allocation reports CC_ERR_OOM)
}

// Row batches [b[i], b[i + 1]) of the n owned rows: equal sizes, the first
// holding every heavy vertex (hubs are the lowest internal ids, so each
// batch's work items are one contiguous range of the pass).
std::vector<int64_t> batch_bounds(const Pass &w, int64_t n, int nb) {
  std::vector<int64_t> b((size_t)nb + 1);
  for (int i = 0; i <= nb; ++i) b[i] = n * i / nb;
  for (int i = 1; i < nb; ++i) b[i] = std::max(b[i], std::min<int64_t>(n, w.max_heavy_v + 1));
  return b;
}

}  // namespace

void run_count(cc_ctx *c, double *X, int dump_table, std::vector<double> *dump, std::vector<double> *root_out,
               const std::vector<int64_t> *dump_rows, TableCache *cache, bool capture) {
  const Plan &pl = c->plan;
  const int k = pl.colours(), elem = c->elem();
  std::fill(c->stats, c->stats + kNStats, 0.0);
  c->stats[10] = c->xmode;
  c->phase_events = c->profiling && c->knobs.phase_events && !capture;
  c->gather_log.clear();
  c->gather_ordinal = 0;
  c->ev_used = 0;
  c->ev_log.clear();
  c->cur_bytes = c->peak_bytes = 0;
  std::fill(c->prof, c->prof + PH_N + 1, 0.0);
  if (pl.k == 1) {  // the single-vertex template maps onto every vertex (any colouring)
    *X = (double)c->n_global;
    return;
  }
  // table rows: owned + halo (halo rows of passive tables land there), or
  // owned only when the exchange is chunked (halo rows go to chunk buffers)
  const int64_t n = c->n_own, rows = c->chunked ? c->n_own : c->n_rows;
  cudaEvent_t t0 = c->ev(), t1 = c->ev();
  if (!capture) CUDA_OK(cudaEventRecord(t0, c->s_main));  // graphs are timed around their launch

  // world > 1: colour-sort the neighbour ranges of both passes (once per
  // colouring); world 1 sorts below, fused with the leaf level (hist)
  if (c->pworld() > 1 && !c->sorted_valid) {
    cudaEvent_t b = c->begin(c->s_main);
    csort(c, c->p_local);
    if (c->xmode == CC_EXCHANGE_RING) {
      for (Pass &w : c->p_peer)
        if (w.items()) csort(c, w);
    } else {
      csort(c, c->p_remote);
    }
    c->end(PH_CSORT, c->s_main, b);
    c->sorted_valid = true;
  }

  // Fused root (world 1): when the root step's neighbour sum N''(P) is needed
  // by no other step, the root is evaluated in the gather's epilogue and
  // N''(P) never reaches HBM.  Mode 2: the root's active part is the lift of
  // the same passive (T_active = N''(P), e.g. two identical subtrees under
  // the root), so the lift is deferred to the root as well.
  const int sr = (int)pl.steps.size() - 1;
  int fuse = 0, defer_lift = -1;
  std::vector<int> last_use(pl.table_last_use);
  {
    const Step &rs = pl.steps[sr];
    if (pl.k == k && !cache && (dump_table < 0 || dump_rows) && c->knobs.fused_root && !c->chunked &&
        c->chunk_cols == 0 && rs.out < 0 && rs.p >= 2) {
      const int P = rs.passive;
      int s_l = -1, users = 0;
      for (int s = 0; s < sr; ++s) {
        if (pl.steps[s].out == rs.active) s_l = s;
        if (pl.steps[s].passive == P) ++users;
      }
      if (rs.a > 1 && s_l >= 0 && pl.steps[s_l].a == 1 && pl.steps[s_l].passive == P && users == 1 &&
          pl.table_last_use[rs.active] == sr) {
        fuse = 2;
        defer_lift = s_l;
        last_use[P] = sr;
      } else if (users == 0 && rs.a > 1) {
        fuse = 1;
      }
    }
  }

  // Fused combine + root (fuse = 3): the root's active table is the output
  // of a combine over the SAME passive (configs[2] and [3]: the legs or
  // subtrees under the root are isomorphic), whose neighbour sum that
  // combine stages anyway -- the root is evaluated in the combine's
  // epilogue and the active table never reaches HBM.
  int fuse_cr = -1;
  bool cr_done = false;
  {
    const Step &rs = pl.steps[sr];
    if (!fuse && pl.k == k && !cache && c->knobs.fused_root && rs.out < 0 && rs.a > 1 && rs.p >= 2 &&
        (dump_table < 0 || (dump_rows && dump_table != rs.active)) && pl.table_last_use[rs.active] == sr) {
      for (int s = 0; s < sr; ++s) {
        const Step &cs = pl.steps[s];
        if (cs.out == rs.active && cs.a >= 2 && cs.passive == rs.passive && c->d_ztab[s] &&
            dev::combine_z_supported(elem, cs.t - 1, cs.a - 1))
          fuse_cr = s;
      }
    }
  }

  const int nt = (int)pl.tables.size();
  int last_hist_use = -1;
  for (int s = 0; s < (int)pl.steps.size(); ++s)
    if (pl.steps[s].p == 1) last_hist_use = s;
  std::vector<int> n_last(pl.n_last_use);

  // Memory plan: when the tables of
  // this plan would not fit the free device memory, the tail of the plan --
  // its last neighbour sum and the row-local steps after it -- runs in row
  // batches, and if even that does not fit, the tail's passive table is
  // never stored but recomputed per batch in column chunks by its combine.
  const MemPlan mp = (cache || (dump_table >= 0 && !dump_rows))
                         ? MemPlan()
                         : plan_memory(c, pl, rows, fuse, defer_lift, fuse_cr, last_hist_use, root_out != nullptr);
  if (mp.tail >= 0) {  // the batched tail evaluates the root per batch (no gather-epilogue root)
    if (fuse == 2) last_use[pl.steps[sr].passive] = pl.table_last_use[pl.steps[sr].passive];
    fuse = 0;
    defer_lift = -1;
    if (mp.rc >= 0) {  // the recomputed table's inputs stay until the end
      const Step &q = pl.steps[mp.rc];
      if (q.active >= 0) last_use[q.active] = sr + 1;
      if (q.p == 1) last_hist_use = sr + 1;
      else n_last[q.passive] = sr + 1;
    }
  }
  if (mp.tail >= 0 && dump_rows && dump_table >= 0) {
    for (int s = mp.tail; s < (int)pl.steps.size(); ++s)
      if (pl.steps[s].out == dump_table || (mp.rc >= 0 && pl.steps[mp.rc].out == dump_table))
        throw Error(CC_ERR_STATE, "the table asked for is produced in the row-batched tail of the memory plan");
  }
  c->stats[12] = mp.tail >= 0 ? mp.nb : 0;
  c->stats[13] = mp.rc >= 0 ? mp.rc_w : 0;

  c->stats[5] = fuse;
  Bufs bufs(c);
  std::vector<int> T(nt, -1), Nb(nt, -1);
  int hist = -1;
  double *per_vertex = nullptr;
  if (root_out || fuse || fuse_cr >= 0 || mp.tail >= 0)
    per_vertex = static_cast<double *>(bufs.ptr(bufs.make((size_t)std::max<int64_t>(n, 1) * 8)));
  if (cache && cache->sorted) {  // an earlier template of this colouring sorted and built the leaf level
    if (last_hist_use >= 0) hist = bufs.alias(cache->hist, cache->hist_bytes);
  } else if (c->pworld() == 1) {  // colour sort + leaf level N''(v, {y}) in one pass over the adjacency
    if (last_hist_use >= 0) {
      const size_t hb = (size_t)rows * c->ld_of(k - 1) * elem;
      if (cache) {
        cache->hist = c->amalloc(hb, c->s_main);
        cache->hist_bytes = hb;
        hist = bufs.alias(cache->hist, hb);
      } else {
        hist = bufs.make(hb);
      }
    }
    cudaEvent_t b = c->begin(c->s_main);
    Pass &p = c->p_full;
    c->stats[3] += dev::launch_csort_hist(elem, p.beg, p.end, c->d_col, c->d_colors, p.view(), k, c->d_col_sorted,
                                          p.goff, p.desc, hist >= 0 ? bufs.ptr(hist) : nullptr, c->ld_of(k - 1), rows,
                                          p.small_from, c->knobs, c->num_sms, c->s_main);
    c->check_launch();
    c->end(PH_CSORT, c->s_main, b);
    c->sorted_valid = true;
    c->stats[1] += (double)p.nnz * 9.0 + (double)p.items() * 64.0 + (hist >= 0 ? (double)n * (k - 1) * elem : 0.0);
    if (hist >= 0) c->stats[0] += (double)c->part.col.size() * k;  // U counts C(k,1) = k colour sets per entry
    if (cache) {
      cache->sorted = true;
      if (!cache->hist) {  // the first template needed no leaf level: build it with the next one that does
        cache->sorted = false;
      }
    }
  }
  // with a cache: the tables this template still has to compute (those not
  // cached, reachable from the root without passing through a cached one)
  std::vector<char> need((size_t)pl.tables.size(), 1);
  std::vector<int> producer((size_t)pl.tables.size(), -1);
  if (cache) {
    for (int s = 0; s < (int)pl.steps.size(); ++s)
      if (pl.steps[s].out >= 0) producer[pl.steps[s].out] = s;
    std::fill(need.begin(), need.end(), 0);
    std::function<void(int)> mark;
    // a passive table is needed only when its neighbour sum is not cached
    auto mark_passive = [&](int id) {
      if (id >= 0 && !cache->tables.count("N" + pl.tables[id].code)) mark(id);
    };
    mark = [&](int id) {
      if (id < 0 || need[id]) return;
      if (cache->tables.count(pl.tables[id].code)) {
        need[id] = 2;  // cached
        return;
      }
      need[id] = 1;
      const Step &ps = pl.steps[producer[id]];
      mark(ps.active);
      mark_passive(ps.passive);
    };
    mark(pl.steps.back().active);
    mark_passive(pl.steps.back().passive);
  }

  auto release_dead = [&](int s) {  // release the tables / neighbour sums whose last use is step s
    if (dump_table >= 0 && !dump_rows) return;
    for (int id = 0; id < nt; ++id) {
      if (T[id] >= 0 && last_use[id] == s) {
        bufs.unref(T[id]);
        T[id] = -1;
      }
      if (Nb[id] >= 0 && n_last[id] == s) {
        bufs.unref(Nb[id]);
        Nb[id] = -1;
      }
    }
    if (hist >= 0 && s == last_hist_use) {
      bufs.unref(hist);
      hist = -2;  // computed and released
    }
  };

  // Sibling pairs (one rank): a narrow passive P2 of a later step whose
  // table is ready -- or is made by a row-local step (its passive the leaf
  // level, its active table alive) that can run now -- is summed in the SAME
  // traversal of the colour-sorted lists as this step's narrow passive (the
  // index stream, colour groups, item setup and N'' row writes paid once).
  // configs[3]: the p = 2 gather takes B3's neighbour sum along (B3 = the
  // (3;2,1) combine, run ahead of its turn).  Off when the tables approach
  // the device size (N''(P2) is allocated earlier than planned).
  std::vector<char> early(pl.steps.size(), 0);  // row-local steps run ahead of their turn
  const bool pair_ok = c->knobs.pair_gather && c->pworld() == 1 && c->chunk_cols == 0 && !cache && mp.tail < 0 &&
                       (dump_table < 0 || dump_rows) &&
                       model_peak(c, pl, rows, fuse, defer_lift, fuse_cr, last_hist_use, root_out != nullptr, mp) <
                           0.4 * c->total_mem;
  auto vecs = [&](int p) { return (int)((binom(k - 1, p - 1) * elem + 15) / 16); };  // 16-byte vectors of a row
  auto pair_partner = [&](int s) -> std::pair<int, int> {  // (step s2 of the sibling, producer to run early or -1)
    const Step &st = pl.steps[s];
    if (!pair_ok || st.p < 2 || vecs(st.p) > 16) return {-1, -1};
    for (int s2 = s + 1; s2 <= sr; ++s2) {
      const Step &q = pl.steps[s2];
      if (q.p < 2 || q.passive == st.passive || Nb[q.passive] >= 0 || pl.n_first_use[q.passive] != s2) continue;
      if ((s2 == sr && fuse) || vecs(st.p) + vecs(q.p) > 24) continue;
      if (T[q.passive] >= 0) return {s2, -1};
      int sp = -1;
      for (int x = s + 1; x < s2; ++x)
        if (pl.steps[x].out == q.passive) sp = x;
      if (sp < 0) continue;
      const Step &ps = pl.steps[sp];
      if (ps.p != 1 || hist < 0 || early[sp] || sp == defer_lift || sp == fuse_cr) continue;
      if (dump_table >= 0 && ps.out == dump_table) continue;  // its sampled rows are copied in its own turn
      if (ps.active >= 0 && T[ps.active] < 0) continue;
      return {s2, sp};
    }
    return {-1, -1};
  };
  auto run_early = [&](int sp) {  // a row-local step over the leaf level, ahead of its turn
    const Step &ps = pl.steps[sp];
    const int Wa = (int)binom(k - 1, ps.a - 1), Wp = k - 1, Wt = (int)binom(k - 1, ps.t - 1);
    early[sp] = 1;
    if (ps.a == 1) {  // lift: T' = N''(leaf)
      T[ps.out] = hist;
      bufs.ref(hist);
      return;
    }
    T[ps.out] = bufs.make((size_t)rows * c->ld_of(Wt) * elem);
    cudaEvent_t b = c->begin(c->s_main);
    c->stats[3] += dev::launch_combine(elem, bufs.ptr(T[ps.active]), c->ld_of(Wa), Wa, bufs.ptr(hist), c->ld_of(Wp), Wp,
                                       c->d_split[sp], (int)binom(ps.t - 1, ps.a - 1), n, bufs.ptr(T[ps.out]),
                                       c->ld_of(Wt), Wt, c->d_ztab[sp], c->zblocks[sp],
                                       (int)zblock_ld(ps.t - 1, ps.a - 1), ps.t - 1, ps.a - 1, c->knobs, c->num_sms,
                                       c->s_main);
    c->check_launch();
    c->end(PH_COMBINE, c->s_main, b);
    c->stats[1] += (double)n * (Wa + Wp + Wt) * elem;
  };

  for (int s = 0; s < (int)pl.steps.size(); ++s) {
    const Step &st = pl.steps[s];
    const int Wa = (int)binom(k - 1, st.a - 1), Wp = (int)binom(k - 1, st.p), Wt = (int)binom(k - 1, st.t - 1);
    if (mp.tail >= 0 && s >= mp.tail) break;  // the batched tail (below)
    if (s == mp.rc) continue;                  // recomputed per batch in column chunks
    if (s == defer_lift) continue;  // T_out = N''(P) is evaluated inside the fused root
    if (early[s]) {  // ran ahead of its turn for a sibling pair
      release_dead(s);
      continue;
    }
    if (cache && st.out >= 0) {
      if (!need[st.out]) continue;  // only feeds tables this template finds cached
      if (need[st.out] == 2) {      // computed by an earlier template of this colouring
        const auto &e = cache->tables[pl.tables[st.out].code];
        T[st.out] = bufs.alias(e.first, e.second);
        ++cache->reused;
        continue;
      }
    }
    if (s == sr && fuse) {
      cc::RootFuse rf;
      rf.mode = fuse;
      rf.A = fuse == 1 ? bufs.ptr(T[st.active]) : nullptr;
      rf.ldA = c->ld_of(Wa);
      rf.WA = Wa;
      rf.per_vertex = per_vertex;
      void *Pp = bufs.ptr(T[st.passive]);
      const int64_t ldP = c->ld_of(binom(k - 1, st.p - 1));
      if (c->pworld() > 1) {
        // partitioned: the fused root needs whole neighbour ranges, so the
        // halo rows of the passive table arrive first and the full ranges
        // are colour-sorted once per colouring (their own buffer)
        if (!c->full_sorted_valid) {
          if (!c->d_col_sorted_full) c->d_col_sorted_full = c->pmalloc<int32_t>(std::max<size_t>(c->part.col.size(), 1));
          c->p_full.col_sorted = c->d_col_sorted_full;
          cudaEvent_t b = c->begin(c->s_main);
          csort(c, c->p_full);
          c->end(PH_CSORT, c->s_main, b);
          c->full_sorted_valid = true;
        }
        comm_after_main(c);
        cudaEvent_t recvd =
            exchange_halo(c, Pp, ldP, 0, ldP, static_cast<char *>(Pp) + (size_t)c->n_own * ldP * elem, ldP);
        CUDA_OK(cudaStreamWaitEvent(c->s_main, recvd, 0));
      }
      gather_pass(c, c->p_full, table_src(Pp, ldP, 0, (int)binom(k - 1, st.p - 1), elem), st.p, nullptr, 0, &rf,
                  c->num_sms);
      cudaEvent_t b = c->begin(c->s_main);
      c->stats[3] += dev::launch_root(8, nullptr, 0, 0, per_vertex, 1, nullptr, n, c->d_partials, c->n_partials,
                                      nullptr, c->d_result, c->s_main);
      c->check_launch();
      c->end(PH_ROOT, c->s_main, b);
      c->stats[1] += (double)n * 8.0;
      break;
    }
    int nbuf;  // buffer of N''
    if (st.p == 1) {
      if (hist < 0) {
        hist = bufs.make((size_t)rows * c->ld_of(k - 1) * elem);
        cudaEvent_t b = c->begin(c->s_main);
        c->stats[3] += dev::launch_hist(elem, c->d_rp, c->d_rp + 1, c->d_col, c->d_colors, c->p_full.view(), n, k,
                                        bufs.ptr(hist), c->ld_of(k - 1), c->num_sms, c->s_main);
        c->check_launch();
        c->end(PH_HIST, c->s_main, b);
        const double nnz = (double)c->part.col.size();
        c->stats[0] += nnz * k;  // U counts C(k,1) = k colour sets per adjacency entry
        c->stats[1] += nnz * 5.0 + (double)n * (k - 1) * elem;
      }
      nbuf = hist;
    } else {
      const int P = st.passive;
      if (Nb[P] < 0) {
        const std::string nkey = cache ? "N" + pl.tables[P].code : std::string();
        if (cache && cache->tables.count(nkey)) {  // neighbour sum of an earlier template
          const auto &e = cache->tables[nkey];
          Nb[P] = bufs.alias(e.first, e.second);
          ++cache->reused;
        } else {
          Nb[P] = bufs.make((size_t)rows * c->ld_of(Wp) * elem);
          const auto pp = pair_partner(s);
          if (pp.first >= 0) {  // one traversal for P and its sibling
            const Step &q = pl.steps[pp.first];
            if (pp.second >= 0) run_early(pp.second);
            const int P2 = q.passive, Win2 = (int)binom(k - 1, q.p - 1);
            Nb[P2] = bufs.make((size_t)rows * c->ld_of(binom(k - 1, q.p)) * elem);
            const PairSrc pr{table_src(bufs.ptr(T[P2]), c->ld_of(Win2), 0, Win2, elem), q.p, bufs.ptr(Nb[P2])};
            const int Win = (int)binom(k - 1, st.p - 1);
            gather_pass(c, c->p_full, table_src(bufs.ptr(T[P]), c->ld_of(Win), 0, Win, elem), st.p, bufs.ptr(Nb[P]), 0,
                        nullptr, c->num_sms, 0, -1, &pr);
            c->stats[15] += 1;  // sibling pairs
          } else {
            aggregate(c, bufs.ptr(T[P]), c->ld_of(binom(k - 1, st.p - 1)), st.p, bufs.ptr(Nb[P]));
          }
          Buf &bb = bufs.pool[Nb[P]];
          if (cache && cache->bytes + bb.bytes <= cache->budget) {
            cache->tables[nkey] = {bb.p, bb.bytes};
            cache->bytes += bb.bytes;
            bb.owned = false;
            ++cache->stored;
          }
        }
      }
      nbuf = Nb[P];
    }
    const int64_t ldN = c->ld_of(Wp);
    if (st.out < 0 && pl.k < k) {  // fewer template vertices than colours: root table, then row sums (Eq. 3)
      int rb = nbuf;  // a = 1: the root table is the neighbour sum itself
      if (st.a > 1) {
        rb = bufs.make((size_t)rows * c->ld_of(Wt) * elem);
        cudaEvent_t b = c->begin(c->s_main);
        c->stats[3] += dev::launch_combine(elem, bufs.ptr(T[st.active]), c->ld_of(Wa), Wa, bufs.ptr(nbuf), ldN, Wp,
                                           c->d_split[s], (int)binom(st.t - 1, st.a - 1), n, bufs.ptr(rb),
                                           c->ld_of(Wt), Wt, c->d_ztab[s], c->zblocks[s],
                                           (int)zblock_ld(st.t - 1, st.a - 1), st.t - 1, st.a - 1, c->knobs,
                                           c->num_sms, c->s_main);
        c->check_launch();
        c->end(PH_COMBINE, c->s_main, b);
        c->stats[1] += (double)n * (Wa + Wp + Wt) * elem;
      }
      cudaEvent_t b = c->begin(c->s_main);
      c->stats[3] += dev::launch_rowsum(elem, bufs.ptr(rb), c->ld_of(Wt), Wt, n, c->d_partials, c->n_partials,
                                        per_vertex, c->d_result, c->s_main);
      c->check_launch();
      c->end(PH_ROOT, c->s_main, b);
      c->stats[1] += (double)n * Wt * elem;
    } else if (st.out < 0 && cr_done) {  // X_v came from the last combine's epilogue: sum over v
      cudaEvent_t b = c->begin(c->s_main);
      c->stats[3] += dev::launch_root(8, nullptr, 0, 0, per_vertex, 1, nullptr, n, c->d_partials, c->n_partials,
                                      nullptr, c->d_result, c->s_main);
      c->check_launch();
      c->end(PH_ROOT, c->s_main, b);
      c->stats[1] += (double)n * 8.0;
    } else if (st.out < 0) {  // root step fused with the sum over v (Eq. 3)
      cudaEvent_t b = c->begin(c->s_main);
      const void *A = st.a > 1 ? bufs.ptr(T[st.active]) : nullptr;
      c->stats[3] += dev::launch_root(elem, A, c->ld_of(Wa), Wa, bufs.ptr(nbuf), ldN, c->d_comp, n, c->d_partials,
                                      c->n_partials, per_vertex, c->d_result, c->s_main);
      c->check_launch();
      c->end(PH_ROOT, c->s_main, b);
      c->stats[1] += (double)n * (st.a > 1 ? 2.0 * Wa : 1.0) * elem;
    } else if (st.a == 1) {  // T'(v, .) = N''(v, .): alias, no kernel
      T[st.out] = nbuf;
      bufs.ref(nbuf);
    } else if (s == fuse_cr &&
               [&] {
                 cudaEvent_t b = c->begin(c->s_main);
                 const int l = dev::launch_combine_root(
                     elem, bufs.ptr(T[st.active]), c->ld_of(Wa), Wa, bufs.ptr(nbuf), ldN, Wp, c->d_ztab[s],
                     c->zblocks[s], (int)zblock_ld(st.t - 1, st.a - 1), st.t - 1, st.a - 1, c->d_comp, n, per_vertex,
                     c->knobs, c->num_sms, c->s_main);
                 if (!l) return false;
                 c->check_launch();
                 c->end(PH_COMBINE, c->s_main, b);
                 c->stats[3] += l;
                 c->stats[1] += (double)n * (Wa + Wp + 1.0) * elem;
                 return true;
               }()) {
      cr_done = true;  // the active table of the root is never stored
      c->stats[5] = 3;
    } else {
      T[st.out] = bufs.make((size_t)rows * c->ld_of(Wt) * elem);
      cudaEvent_t b = c->begin(c->s_main);
      c->stats[3] += dev::launch_combine(elem, bufs.ptr(T[st.active]), c->ld_of(Wa), Wa, bufs.ptr(nbuf), ldN, Wp,
                                         c->d_split[s], (int)binom(st.t - 1, st.a - 1), n, bufs.ptr(T[st.out]),
                                         c->ld_of(Wt), Wt, c->d_ztab[s], c->zblocks[s],
                                         (int)zblock_ld(st.t - 1, st.a - 1), st.t - 1, st.a - 1, c->knobs,
                                         c->num_sms, c->s_main);
      c->check_launch();
      c->end(PH_COMBINE, c->s_main, b);
      c->stats[1] += (double)n * (Wa + Wp + Wt) * elem;
    }
    if (cache && st.out >= 0 && T[st.out] >= 0 && bufs.pool[T[st.out]].owned &&
        !cache->tables.count(pl.tables[st.out].code) &&
        cache->bytes + bufs.pool[T[st.out]].bytes <= cache->budget) {  // keep it for the next templates
      Buf &bb = bufs.pool[T[st.out]];
      cache->tables[pl.tables[st.out].code] = {bb.p, bb.bytes};
      cache->bytes += bb.bytes;
      bb.owned = false;
      ++cache->stored;
    }
    if (dump_rows && st.out == dump_table && st.out >= 0 && T[st.out] >= 0) {  // sampled rows of this table
      const int W = (int)binom(k - 1, pl.tables[dump_table].size - 1);
      const size_t ld = (size_t)c->ld_of(W);
      std::vector<char> raw(dump_rows->size() * (size_t)W * elem);
      for (size_t i = 0; i < dump_rows->size(); ++i)
        CUDA_OK(cudaMemcpyAsync(raw.data() + i * W * elem,
                                static_cast<char *>(bufs.ptr(T[st.out])) + (size_t)(*dump_rows)[i] * ld * elem,
                                (size_t)W * elem, cudaMemcpyDeviceToHost, c->s_main));
      CUDA_OK(cudaStreamSynchronize(c->s_main));
      dump->assign(dump_rows->size() * (size_t)W, 0.0);
      for (size_t i = 0; i < dump->size(); ++i)
        (*dump)[i] = elem == 8 ? reinterpret_cast<double *>(raw.data())[i] : reinterpret_cast<float *>(raw.data())[i];
    }
    release_dead(s);
  }
  if (mp.tail >= 0) {
    // The batched tail (memory plan): for each batch of rows [r0, r1), the
    // neighbour sum of step g for those rows only (their work items), from
    // the stored passive table or from its column chunks recomputed by their
    // combine for every row, then the row-local steps g..root on those rows.
    const int g = mp.tail;
    const Step &gs = pl.steps[g];
    const int P = gs.passive;
    const int WinP = (int)binom(k - 1, gs.p - 1), WpP = (int)binom(k - 1, gs.p);
    const int64_t ldP = c->ld_of(WinP), ldNP = c->ld_of(WpP);
    Pass &w = c->p_full;
    const std::vector<int64_t> bounds = batch_bounds(w, n, mp.nb);
    int rcb = -1;
    const int64_t ldw = mp.rc >= 0 ? c->ld_of(mp.rc_w) : 0;
    if (mp.rc >= 0) rcb = bufs.make((size_t)std::max<int64_t>(rows, 1) * ldw * elem);
    for (size_t b = 0; b + 1 < bounds.size(); ++b) {
      const int64_t r0 = bounds[b], r1 = bounds[b + 1], nr = r1 - r0;
      if (nr <= 0) continue;
      // the batch's work items: its light vertices (contiguous in the item
      // list) and, in batch 0, every heavy segment
      const int64_t lo = std::lower_bound(w.light_h.begin(), w.light_h.end(), (int32_t)r0) - w.light_h.begin();
      const int64_t hi = std::lower_bound(w.light_h.begin(), w.light_h.end(), (int32_t)r1) - w.light_h.begin();
      const int64_t from = b == 0 ? 0 : w.n_seg + lo, to = w.n_seg + hi;
      // row r0 of every table the tail reads: stored in full (offset) or made in this batch
      std::vector<const void *> TB(nt, nullptr), NB(nt, nullptr);
      std::vector<int> batch_bufs;
      auto row0 = [&](int buf, int64_t ld) -> const void * {
        return static_cast<const char *>(bufs.ptr(buf)) + (size_t)r0 * ld * elem;
      };
      const int nbb = bufs.make((size_t)nr * ldNP * elem);
      batch_bufs.push_back(nbb);
      NB[P] = bufs.ptr(nbb);
      void *Nv = static_cast<char *>(bufs.ptr(nbb)) - (size_t)r0 * ldNP * elem;  // row v at Nv + v ldNP
      if (mp.rc < 0) {
        gather_pass(c, w, table_src(bufs.ptr(T[P]), ldP, 0, WinP, elem), gs.p, Nv, 0, nullptr, c->num_sms, from, to);
      } else {
        const Step &q = pl.steps[mp.rc];
        const int qa = (int)binom(k - 1, q.a - 1), qp = (int)binom(k - 1, q.p);
        const void *Aq = bufs.ptr(T[q.active]);
        const void *Nq = q.p == 1 ? bufs.ptr(hist) : bufs.ptr(Nb[q.passive]);
        const auto chunks = column_chunks(WinP, mp.rc_w);
        for (size_t i = 0; i < chunks.size(); ++i) {
          const int c0 = chunks[i].first, cw = chunks[i].second;
          // columns [c0, c0 + cw) of the passive table, every row: column o of row v at outv + v ldw + o
          void *outv = static_cast<char *>(bufs.ptr(rcb)) - (size_t)c0 * elem;
          cudaEvent_t e = c->begin(c->s_main);
          c->stats[3] += dev::launch_combine_cols(elem, Aq, c->ld_of(qa), qa, Nq, c->ld_of(qp), qp, c->d_split[mp.rc],
                                                  (int)binom(q.t - 1, q.a - 1), n, outv, ldw, WinP, c0, c0 + cw,
                                                  c->knobs, c->num_sms, c->s_main);
          c->check_launch();
          c->end(PH_COMBINE, c->s_main, e);
          c->stats[1] += (double)n * (qa + qp + cw) * elem;
          gather_pass(c, w, Src{bufs.ptr(rcb), ldw, c0, cw}, gs.p, Nv, i > 0, nullptr, c->num_sms, from, to);
        }
      }
      double *pv = per_vertex + r0;
      bool cr_batch = false;
      for (int s2 = g; s2 <= sr; ++s2) {
        const Step &st = pl.steps[s2];
        const int Wa = (int)binom(k - 1, st.a - 1), Wp = (int)binom(k - 1, st.p), Wt = (int)binom(k - 1, st.t - 1);
        const int64_t ldA = c->ld_of(Wa), ldN = c->ld_of(Wp), ldT = c->ld_of(Wt);
        const void *A = st.active < 0 ? nullptr : (TB[st.active] ? TB[st.active] : row0(T[st.active], ldA));
        const void *Nn = st.p == 1 ? row0(hist, c->ld_of(k - 1))
                                   : (NB[st.passive] ? NB[st.passive] : row0(Nb[st.passive], ldN));
        cudaEvent_t e = c->begin(c->s_main);
        if (st.out < 0 && pl.k < k) {  // fewer template vertices than colours: root table, row sums
          const void *R = Nn;
          if (st.a > 1) {
            const int rb = bufs.make((size_t)nr * ldT * elem);
            batch_bufs.push_back(rb);
            c->stats[3] += dev::launch_combine(elem, A, ldA, Wa, Nn, ldN, Wp, c->d_split[s2],
                                               (int)binom(st.t - 1, st.a - 1), nr, bufs.ptr(rb), ldT, Wt,
                                               c->d_ztab[s2], c->zblocks[s2], (int)zblock_ld(st.t - 1, st.a - 1),
                                               st.t - 1, st.a - 1, c->knobs, c->num_sms, c->s_main);
            R = bufs.ptr(rb);
          }
          c->stats[3] += dev::launch_rowsum(elem, R, ldT, Wt, nr, c->d_partials, c->n_partials, pv, c->d_result,
                                            c->s_main);
        } else if (st.out < 0 && !cr_batch && !cr_done) {  // the root on these rows (X_v into per_vertex)
          c->stats[3] += dev::launch_root(elem, A, ldA, Wa, Nn, ldN, c->d_comp, nr, c->d_partials, c->n_partials, pv,
                                          c->d_result, c->s_main);
        } else if (st.out < 0) {
          // X_v came from the combine's epilogue (fused mode 3)
        } else if (st.a == 1) {
          TB[st.out] = Nn;  // the lift is the neighbour sum itself
        } else if (s2 == fuse_cr &&
                   (cr_batch = dev::launch_combine_root(elem, A, ldA, Wa, Nn, ldN, Wp, c->d_ztab[s2], c->zblocks[s2],
                                                        (int)zblock_ld(st.t - 1, st.a - 1), st.t - 1, st.a - 1,
                                                        c->d_comp, nr, pv, c->knobs, c->num_sms, c->s_main) > 0)) {
          c->stats[3] += 1;
          c->stats[5] = 3;
        } else {
          const int ob = bufs.make((size_t)nr * ldT * elem);
          batch_bufs.push_back(ob);
          TB[st.out] = bufs.ptr(ob);
          c->stats[3] += dev::launch_combine(elem, A, ldA, Wa, Nn, ldN, Wp, c->d_split[s2],
                                             (int)binom(st.t - 1, st.a - 1), nr, bufs.ptr(ob), ldT, Wt, c->d_ztab[s2],
                                             c->zblocks[s2], (int)zblock_ld(st.t - 1, st.a - 1), st.t - 1, st.a - 1,
                                             c->knobs, c->num_sms, c->s_main);
        }
        c->check_launch();
        c->end(st.out < 0 ? PH_ROOT : PH_COMBINE, c->s_main, e);
        c->stats[1] += (double)nr * (Wa + Wp + (st.out < 0 ? 1 : Wt)) * elem;
      }
      for (int bb : batch_bufs) bufs.unref(bb);
    }
    // X = sum of X_v over every row, in a fixed order
    cudaEvent_t e = c->begin(c->s_main);
    c->stats[3] += dev::launch_root(8, nullptr, 0, 0, per_vertex, 1, nullptr, n, c->d_partials, c->n_partials,
                                    nullptr, c->d_result, c->s_main);
    c->check_launch();
    c->end(PH_ROOT, c->s_main, e);
  }
  if (c->pworld() > 1) {
    cudaEvent_t b = c->begin(c->s_main);
    if (c->loop) loopback_allreduce(c, c->d_result, 1, c->s_main);
    else NCCL_OK(nccl().AllReduce(c->d_result, c->d_result, 1, ncclFloat64, ncclSum, c->comm, c->s_main));
    c->end(PH_EXCHANGE, c->s_main, b);
  }
  if (!capture) CUDA_OK(cudaEventRecord(t1, c->s_main));
  if (capture) {  // a CUDA graph of the count's device work (use_graphs): no host copies, no syncs
    for (auto &b : bufs.pool)
      if (b.p && b.owned) c->afree(b.p, b.bytes, c->s_main);
    c->stats[4] = (double)c->peak_bytes;
    return;
  }
  double host_x = 0;
  CUDA_OK(cudaMemcpyAsync(&host_x, c->d_result, sizeof(double), cudaMemcpyDeviceToHost, c->s_main));
  if (dump && !dump_rows && dump_table >= 0 && T[dump_table] >= 0) {
    const int W = (int)binom(k - 1, pl.tables[dump_table].size - 1);
    std::vector<char> raw((size_t)n * c->ld_of(W) * elem);
    if (!raw.empty())
      CUDA_OK(cudaMemcpyAsync(raw.data(), bufs.ptr(T[dump_table]), raw.size(), cudaMemcpyDeviceToHost, c->s_main));
    CUDA_OK(cudaStreamSynchronize(c->s_main));
    dump->assign((size_t)n * W, 0.0);
    for (int64_t v = 0; v < n; ++v)
      for (int j = 0; j < W; ++j) {
        const size_t off = (size_t)v * c->ld_of(W) + j;
        (*dump)[(size_t)v * W + j] =
            elem == 8 ? reinterpret_cast<double *>(raw.data())[off] : reinterpret_cast<float *>(raw.data())[off];
      }
  }
  if (root_out) {
    root_out->resize((size_t)n);
    if (n) CUDA_OK(cudaMemcpyAsync(root_out->data(), per_vertex, (size_t)n * 8, cudaMemcpyDeviceToHost, c->s_main));
  }
  for (auto &b : bufs.pool)
    if (b.p && b.owned) c->afree(b.p, b.bytes, c->s_main);
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  if (c->pworld() > 1) CUDA_OK(cudaStreamSynchronize(c->s_comm));
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, t0, t1));
  c->prof[0] = ms;
  std::vector<float> ev_ms(c->ev_log.size(), 0.f);
  for (size_t i = 0; i < c->ev_log.size(); ++i) {
    auto &e = c->ev_log[i];
    CUDA_OK(cudaEventElapsedTime(&ev_ms[i], e.second.first, e.second.second));
    c->prof[1 + e.first] += ev_ms[i];
  }
  // the longest gather launch (the dominant kernel): its algorithmic bytes, ms
  // and 1-based ordinal among the count's neighbour-sum passes
  for (size_t i = 0; i < c->gather_log.size(); ++i) {
    const auto &g = c->gather_log[i];
    if (ev_ms[g.first] > c->stats[7]) {
      c->stats[6] = g.second;
      c->stats[7] = ev_ms[g.first];
      c->stats[14] = (double)(i + 1);
    }
  }
  c->stats[8] = (double)c->gather_log.size();
  c->stats[4] = (double)c->peak_bytes;
  if (!std::isfinite(host_x)) throw Error(CC_ERR_NONFINITE, "colourful count is not finite (fp32 table overflow?)");
  *X = host_x;
}

}  // namespace cc

namespace cc {

// One count through a CUDA graph of its device work (cc_options.use_graphs,
// one rank): captured on the first call and after any change of graph,
// template, knobs or profiling (c->epoch), replayed otherwise -- the
// colouring is data, so a new one replays the same graph.
void count_graph(cc_ctx *c, double *X) {
  if (!c->graph_ev[0]) {
    CUDA_OK(cudaEventCreate(&c->graph_ev[0]));
    CUDA_OK(cudaEventCreate(&c->graph_ev[1]));
  }
  if (!c->gexec || c->gepoch != c->epoch) {
    if (c->gexec) {
      CUDA_OK(cudaStreamSynchronize(c->s_main));
      cudaGraphExecDestroy(c->gexec);
      c->gexec = nullptr;
    }
    CUDA_OK(cudaStreamBeginCapture(c->s_main, cudaStreamCaptureModeRelaxed));
    cudaGraph_t g = nullptr;
    try {
      run_count(c, X, -1, nullptr, nullptr, nullptr, nullptr, true);
    } catch (...) {
      cudaStreamEndCapture(c->s_main, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CUDA_OK(cudaStreamEndCapture(c->s_main, &g));
    const cudaError_t e = cudaGraphInstantiate(&c->gexec, g, 0);
    cudaGraphDestroy(g);
    CUDA_OK(e);
    c->gepoch = c->epoch;
  }
  CUDA_OK(cudaEventRecord(c->graph_ev[0], c->s_main));
  CUDA_OK(cudaGraphLaunch(c->gexec, c->s_main));
  CUDA_OK(cudaEventRecord(c->graph_ev[1], c->s_main));
  double host_x = 0;
  CUDA_OK(cudaMemcpyAsync(&host_x, c->d_result, sizeof(double), cudaMemcpyDeviceToHost, c->s_main));
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, c->graph_ev[0], c->graph_ev[1]));
  std::fill(c->prof, c->prof + PH_N + 1, 0.0);
  c->prof[0] = ms;
  if (!std::isfinite(host_x)) throw Error(CC_ERR_NONFINITE, "colourful count is not finite (fp32 table overflow?)");
  *X = host_x;
}

std::vector<double> run_iterations(cc_ctx *c, int iterations, uint64_t seed0) {
  std::vector<double> xs((size_t)iterations, 0.0);
  const bool rep = c->opt.replicas && c->opt.world > 1;
  for (int j = 0; j < iterations; ++j) {
    if (rep && j % c->opt.world != c->opt.rank) continue;
    launch_colouring(c, seed0 + (uint64_t)j);
    if (c->opt.use_graphs && c->pworld() == 1) count_graph(c, &xs[j]);
    else run_count(c, &xs[j], -1, nullptr, nullptr);
  }
  if (rep) {  // every rank ends with every X_j (the others' entries are 0 here)
    double *d = static_cast<double *>(c->amalloc((size_t)iterations * 8, c->s_main));
    CUDA_OK(cudaMemcpyAsync(d, xs.data(), (size_t)iterations * 8, cudaMemcpyHostToDevice, c->s_main));
    if (c->loop) loopback_allreduce(c, d, (size_t)iterations, c->s_main);
    else NCCL_OK(nccl().AllReduce(d, d, (size_t)iterations, ncclFloat64, ncclSum, c->comm, c->s_main));
    CUDA_OK(cudaMemcpyAsync(xs.data(), d, (size_t)iterations * 8, cudaMemcpyDeviceToHost, c->s_main));
    c->afree(reinterpret_cast<void *&>(d), (size_t)iterations * 8, c->s_main);
    CUDA_OK(cudaStreamSynchronize(c->s_main));
  }
  return xs;
}

}  // namespace cc
