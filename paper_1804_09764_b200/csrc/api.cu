// api.cu -- the C ABI of include/cc.h: argument checks, state machine,
// error conversion (no C++ exception crosses the boundary).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "ctx.h"

using cc::Error;

namespace {

cc_status fail(cc_ctx *c, const Error &e) {
  if (c) {
    c->err = e.what();
    if (e.status == CC_ERR_CUDA || e.status == CC_ERR_NCCL) c->poisoned = true;
  }
  return e.status;
}

#define API_BEGIN(c)                                             \
  if (!(c)) return CC_ERR_ARG;                                   \
  if ((c)->poisoned) {                                           \
    (c)->err = "context poisoned by an earlier CUDA/NCCL error"; \
    return CC_ERR_STATE;                                         \
  }                                                              \
  try {                                                          \
    CUDA_OK(cudaSetDevice((c)->opt.device));
#define API_END(c)                         \
  }                                        \
  catch (const Error &e) {                 \
    return fail((c), e);                   \
  }                                        \
  catch (const std::bad_alloc &) {         \
    (c)->err = "host allocation failed";   \
    return CC_ERR_OOM;                     \
  }                                        \
  catch (const std::exception &e) {        \
    (c)->err = e.what();                   \
    return CC_ERR_ARG;                     \
  }                                        \
  (c)->err.clear();                        \
  return CC_OK;

void free_persistent(cc_ctx *c) {
  for (void *p : c->persistent) cudaFree(p);
  c->persistent.clear();
  c->d_rp = c->d_mid = nullptr;
  c->d_col = c->d_col_sorted = c->d_orig = c->d_send_idx = nullptr;
  c->d_colors = nullptr;
  c->p_full = c->p_local = c->p_remote = cc::Pass();
  c->p_peer.clear();
  c->xmode = 0;
  c->d_split.clear();
  c->d_ztab.clear();
  c->zblocks.clear();
  c->d_map.clear();
  c->d_skip.clear();
  c->skip_words.clear();
  c->d_comp = nullptr;
  c->d_partials = c->d_result = nullptr;
  c->d_arrive = nullptr;
  c->arrive_cap = 0;
  c->max_hv = c->max_seg = 0;
  c->has_graph = c->has_colors = c->sorted_valid = c->full_sorted_valid = false;
  c->d_col_sorted_full = nullptr;
}

void alloc_scratch(cc_ctx *c) {
  c->n_partials = cc::dev::root_partials_blocks(c->num_sms);
  c->d_partials = c->pmalloc<double>((size_t)c->n_partials);
  c->d_result = c->pmalloc<double>(1);
}

// Implementation knobs by name.
int *knob_ptr(cc::dev::Knobs &k, const std::string &name) {
  if (name == "fused_root") return &k.fused_root;
  if (name == "sector_skip") return &k.sector_skip;
  if (name == "gather_impl") return &k.gather_impl;
  if (name == "narrow_impl") return &k.narrow_impl;
  if (name == "narrow_split") return &k.narrow_split;
  if (name == "csort_small") return &k.csort_small;
  if (name == "combine_impl") return &k.combine_impl;
  if (name == "acc32") return &k.acc32;
  if (name == "phase_events") return &k.phase_events;
  if (name == "hub_l2_pct") return &k.hub_l2_pct;
  if (name == "grid_reserve") return &k.grid_reserve;
  if (name == "tail_batches") return &k.tail_batches;
  if (name == "layout") return &k.layout;
  if (name == "lean_split") return &k.lean_split;
  if (name == "short_lists") return &k.short_lists;
  if (name == "short_split") return &k.short_split;
  if (name == "rows_variant") return &k.rows_variant;
  if (name == "pair_gather") return &k.pair_gather;
  if (name == "combine_wreg") return &k.combine_wreg;
  if (name == "combine_static") return &k.combine_static;
  if (name == "combine_zglobal") return &k.combine_zglobal;
  if (name == "wide_warps") return &k.wide_warps;
  if (name == "wide_nv") return &k.wide_nv;
  if (name == "tail_warps") return &k.tail_warps;
  if (name == "nvtx_mark") return &k.nvtx_mark;
  if (name == "tail_recompute_cols") return &k.tail_recompute_cols;
  return nullptr;
}

// CC_<NAME> from the environment, read once per context
void knobs_from_env(cc::dev::Knobs &k) {
  static const char *names[] = {"fused_root", "sector_skip", "gather_impl", "narrow_impl", "narrow_split",
                                "csort_small", "combine_impl", "acc32", "phase_events", "hub_l2_pct", "grid_reserve",
                                "tail_batches", "tail_recompute_cols", "layout", "nvtx_mark", "lean_split", "short_lists", "short_split", "rows_variant",
                                "pair_gather", "combine_wreg", "combine_static", "combine_zglobal", "wide_warps", "wide_nv", "tail_warps"};
  for (const char *n : names) {
    std::string env = "CC_";
    for (const char *q = n; *q; ++q) env += (char)std::toupper((unsigned char)*q);
    if (const char *v = std::getenv(env.c_str())) *knob_ptr(k, n) = std::atoi(v);
  }
}

// dense colex index (k-universe) -> compressed index of the row of colour c
// (DESIGN.md "Data layout"); -1 if the set does not contain c
int64_t compressed_index(uint32_t S, int c) {
  if (!(S >> c & 1u)) return -1;
  return cc::colex_rank(cc::squeeze(S & ~(1u << c), c));
}

}  // namespace

extern "C" {

cc_status cc_default_options(cc_options *opt) {
  if (!opt) return CC_ERR_ARG;
  std::memset(opt, 0, sizeof(*opt));
  opt->precision = CC_FP64;
  opt->world = 1;
  opt->use_graphs = 0;
  opt->relabel_seed = 0x5eed;
  return CC_OK;
}

cc_status cc_loopback_create(int32_t world, void **group) {
  if (world < 1 || world > 64 || !group) return CC_ERR_ARG;
  *group = new cc::LoopbackGroup(world);
  return CC_OK;
}

void cc_loopback_destroy(void *group) { delete static_cast<cc::LoopbackGroup *>(group); }

cc_status cc_nccl_unique_id(void *out128) {
  if (!out128) return CC_ERR_ARG;
  auto &api = cc::nccl();
  if (!api.ok) return CC_ERR_NCCL;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return CC_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return CC_OK;
}

cc_status cc_nccl_device_selftest(int32_t device) { return cc::device_selftest(device); }

cc_status cc_nccl_selftest(int32_t device) {
  auto &api = cc::nccl();
  if (!api.ok) return CC_ERR_NCCL;
  ncclComm_t comm = nullptr;
  cudaStream_t s = nullptr;
  double *d = nullptr;
  cc_status st = CC_OK;
  try {
    CUDA_OK(cudaSetDevice(device));
    ncclUniqueId id;
    NCCL_OK(api.GetUniqueId(&id));
    NCCL_OK(api.CommInitRank(&comm, 1, id, 0));
    CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CUDA_OK(cudaMalloc(&d, 4 * sizeof(double)));
    const double h0[4] = {1.5, 0.0, 0.0, -2.25};
    CUDA_OK(cudaMemcpyAsync(d, h0, sizeof(h0), cudaMemcpyHostToDevice, s));
    // the calls of the halo exchange (a grouped send/recv, here to itself)
    // and of the final reduction, with the same argument types
    NCCL_OK(api.GroupStart());
    NCCL_OK(api.Send(d, 1, ncclFloat64, 0, comm, s));
    NCCL_OK(api.Recv(d + 1, 1, ncclFloat64, 0, comm, s));
    NCCL_OK(api.GroupEnd());
    NCCL_OK(api.AllReduce(d + 3, d + 2, 1, ncclFloat64, ncclSum, comm, s));
    double h[4];
    CUDA_OK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (h[1] != 1.5 || h[2] != -2.25) st = CC_ERR_NCCL;
  } catch (const Error &e) {
    st = e.status;
  }
  if (d) cudaFree(d);
  if (s) cudaStreamDestroy(s);
  if (comm) api.CommDestroy(comm);
  return st;
}

cc_status cc_create(const cc_options *opt, cc_ctx **out) {
  if (!opt || !out) return CC_ERR_ARG;
  if (opt->precision != CC_FP64 && opt->precision != CC_FP32) return CC_ERR_ARG;
  if (opt->world < 1 || opt->world > 64 || opt->rank < 0 || opt->rank >= opt->world) return CC_ERR_ARG;
  if (opt->world > 1 && !opt->nccl_id && !opt->loopback) return CC_ERR_ARG;
  if (opt->chunk_cols < 0 || opt->segment_len < 0 || opt->use_graphs < 0 || opt->use_graphs > 1) return CC_ERR_ARG;
  if (opt->replicas < 0 || opt->replicas > 1) return CC_ERR_ARG;
  if (opt->exchange < CC_EXCHANGE_AUTO || opt->exchange > CC_EXCHANGE_DEVICE) return CC_ERR_ARG;
  if (opt->exchange == CC_EXCHANGE_DEVICE && opt->loopback) return CC_ERR_ARG;
  std::unique_ptr<cc_ctx> c(new cc_ctx());
  c->opt = *opt;
  c->opt.nccl_id = nullptr;
  c->chunk_cols = opt->chunk_cols;
  knobs_from_env(c->knobs);
  try {
    CUDA_OK(cudaSetDevice(opt->device));
    CUDA_OK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, opt->device));
    int l2 = 0;
    CUDA_OK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, opt->device));
    if (l2 > 0) c->l2_bytes = l2;
    {
      size_t fr = 0, tot = 0;
      CUDA_OK(cudaMemGetInfo(&fr, &tot));
      c->total_mem = (double)tot;
    }
    CUDA_OK(cudaStreamCreateWithFlags(&c->s_main, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, opt->device));
    uint64_t thr = UINT64_MAX;
    CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    alloc_scratch(c.get());
    if (opt->world > 1 && opt->loopback) {
      c->loop = static_cast<cc::LoopbackGroup *>(opt->loopback);
      if (c->loop->world != opt->world) throw Error(CC_ERR_ARG, "loopback group size != world");
    } else if (opt->world > 1) {
      auto &api = cc::nccl();
      if (!api.ok) throw Error(CC_ERR_NCCL, api.why);
      ncclUniqueId id;
      std::memcpy(&id, opt->nccl_id, sizeof(id));
      NCCL_OK(api.CommInitRank(&c->comm, opt->world, id, opt->rank));
    }
  } catch (const Error &e) {
    if (c->s_main) cudaStreamDestroy(c->s_main);
    if (c->s_comm) cudaStreamDestroy(c->s_comm);
    for (void *p : c->persistent) cudaFree(p);
    return e.status;
  }
  *out = c.release();
  return CC_OK;
}

void cc_destroy(cc_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->opt.device);
  if (c->s_main) cudaStreamSynchronize(c->s_main);
  if (c->s_comm) cudaStreamSynchronize(c->s_comm);
  cc::devx_free(c);
  if (c->comm) cc::nccl().CommDestroy(c->comm);
  for (void *p : c->persistent) cudaFree(p);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  for (auto e : c->graph_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_color)
    if (e) cudaEventDestroy(e);
  if (c->s_main) cudaStreamDestroy(c->s_main);
  if (c->s_comm) cudaStreamDestroy(c->s_comm);
  {  // hand the stream-ordered pool's cached blocks back to the device
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c->opt.device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  delete c;
}

const char *cc_last_error(const cc_ctx *c) { return c ? c->err.c_str() : "null context"; }

cc_status cc_load_graph(cc_ctx *c, int64_t n, const int64_t *row_ptr, const int32_t *col) {
  API_BEGIN(c)
  cc::HostGraph g = cc::validate_graph(n, row_ptr, col);
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  free_persistent(c);
  alloc_scratch(c);
  cc::load_graph(c, g);
  if (c->has_template) cc::replan(c, false);
  API_END(c)
}

cc_status cc_set_template(cc_ctx *c, int32_t k, const int32_t *parent) { return cc_set_template_colors(c, k, parent, k); }

cc_status cc_set_template_colors(cc_ctx *c, int32_t k, const int32_t *parent, int32_t colours) {
  API_BEGIN(c)
  cc::make_plan(k, parent);  // validates (throws CC_ERR_TEMPLATE)
  if (colours < k || colours > cc::kMaxK) throw Error(CC_ERR_ARG, "colours must be in [k, 16]");
  c->user_parent.assign(parent, parent + k);
  c->user_kc = colours;
  c->has_colors = false;
  c->sorted_valid = c->full_sorted_valid = false;
  cc::replan(c, false);
  c->has_template = true;
  API_END(c)
}

cc_status cc_color(cc_ctx *c, uint64_t seed) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_color needs a graph and a template");
  cc::launch_colouring(c, seed);
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, c->ev_color[0], c->ev_color[1]));
  c->color_ms = ms;
  API_END(c)
}

cc_status cc_set_colors(cc_ctx *c, const uint8_t *colors) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_set_colors needs a graph and a template");
  if (!colors && c->n_global) throw Error(CC_ERR_ARG, "colors is NULL");
  // one H2D copy of the caller's array (DMA when it is pinned), then the
  // permutation to the internal row order and the range check on the device
  unsigned bad = 0;
  if (c->n_global) {
    CUDA_OK(cudaMemsetAsync(c->d_bad, 0, sizeof(unsigned), c->s_main));
    CUDA_OK(cudaMemcpyAsync(c->d_color_stage, colors, (size_t)c->n_global, cudaMemcpyHostToDevice, c->s_main));
    cc::dev::launch_permute_colors(c->d_color_stage, c->d_orig, c->n_crow, c->plan.colours(), c->d_colors, c->d_bad,
                                   c->s_main);
    c->check_launch();
    CUDA_OK(cudaMemcpyAsync(&bad, c->d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, c->s_main));
  }
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  if (bad) throw Error(CC_ERR_ARG, "colour out of [0, k)");
  c->has_colors = true;
  c->sorted_valid = c->full_sorted_valid = false;
  API_END(c)
}

cc_status cc_get_colors(cc_ctx *c, uint8_t *colors) {
  API_BEGIN(c)
  if (!c->has_colors) throw Error(CC_ERR_STATE, "no colouring");
  if (c->pworld() != 1) throw Error(CC_ERR_STATE, "cc_get_colors needs the whole graph on this rank");
  std::vector<uint8_t> h((size_t)c->n_crow);
  if (!h.empty()) CUDA_OK(cudaMemcpy(h.data(), c->d_colors, h.size(), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < c->part.n_own; ++i) colors[c->part.own_orig[i]] = h[i];
  for (size_t i = 0; i < c->part.iso_orig.size(); ++i) colors[c->part.iso_orig[i]] = h[c->n_rows + i];
  API_END(c)
}

cc_status cc_count_colorful(cc_ctx *c, double *X) {
  API_BEGIN(c)
  if (!X) throw Error(CC_ERR_ARG, "output pointer is NULL");
  if (!c->has_graph || !c->has_template || !c->has_colors)
    throw Error(CC_ERR_STATE, "cc_count_colorful needs a graph, a template and a colouring");
  if (c->opt.use_graphs && c->pworld() == 1) cc::count_graph(c, X);
  else cc::run_count(c, X, -1, nullptr, nullptr);
  API_END(c)
}

cc_status cc_count_colorful_multi(cc_ctx *c, int32_t n_templates, const int32_t *sizes, const int32_t *parents,
                                  double *X) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template || !c->has_colors)
    throw Error(CC_ERR_STATE, "cc_count_colorful_multi needs a graph, a template and a colouring");
  if (c->pworld() != 1) throw Error(CC_ERR_STATE, "cc_count_colorful_multi needs the whole graph on this rank");
  if (n_templates < 0 || (n_templates && (!sizes || !parents || !X))) throw Error(CC_ERR_ARG, "bad template list");
  const int kc = c->plan.colours();
  int64_t off = 0;
  for (int i = 0; i < n_templates; ++i) {
    if (sizes[i] < 1 || sizes[i] > kc) throw Error(CC_ERR_ARG, "template larger than the colouring's colours");
    cc::make_plan(sizes[i], parents + off);  // validates (CC_ERR_TEMPLATE)
    off += sizes[i];
  }
  const std::vector<int32_t> saved(c->user_parent);
  const int saved_kc = c->user_kc;
  struct Restore {
    cc_ctx *c;
    const std::vector<int32_t> &parent;
    int kc;
    cc::TableCache cache;
    ~Restore() {
      try {
        cc::free_cache(c, cache);
        c->user_parent = parent;
        c->user_kc = kc;
        cc::replan(c, false);
      } catch (...) {
      }
    }
  } restore{c, saved, saved_kc, {}};
  size_t free_b = 0, total_b = 0;
  CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
  restore.cache.budget = free_b / 4;  // shared tables kept while they fit a quarter of the free memory
  c->user_kc = kc;
  off = 0;
  for (int i = 0; i < n_templates; ++i) {
    c->user_parent.assign(parents + off, parents + off + sizes[i]);
    off += sizes[i];
    cc::replan(c, false);
    cc::run_count(c, &X[i], -1, nullptr, nullptr, nullptr, &restore.cache);
  }
  c->stats[9] = (double)restore.cache.reused;  // (reported through cc_last_stats out[9] for this call)
  API_END(c)
}

cc_status cc_estimate(cc_ctx *c, int32_t iterations, uint64_t seed0, double *estimate, double *per_iter) {
  API_BEGIN(c)
  if (iterations < 1 || !estimate) throw Error(CC_ERR_ARG, "iterations >= 1 and estimate != NULL required");
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_estimate needs a graph and a template");
  const std::vector<double> xs = cc::run_iterations(c, iterations, seed0);
  long double mean = 0;
  for (double x : xs) mean += x;
  mean /= iterations;
  // 1 / P(a map is colourful) = kc^k (kc-k)! / kc! (PAPER.md line 146 with kc colours)
  long double scale = 1;
  for (int i = 0; i < c->plan.k; ++i) scale *= (long double)c->plan.colours() / (c->plan.colours() - i);
  *estimate = (double)(mean * scale / (long double)c->plan.aut);
  if (per_iter) std::copy(xs.begin(), xs.end(), per_iter);
  API_END(c)
}

cc_status cc_estimate_mom(cc_ctx *c, int32_t iterations, uint64_t seed0, int32_t groups, double *estimate,
                          double *per_iter) {
  API_BEGIN(c)
  if (iterations < 1 || groups < 1 || groups > iterations || !estimate)
    throw Error(CC_ERR_ARG, "need 1 <= groups <= iterations and estimate != NULL");
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_estimate_mom needs a graph and a template");
  const std::vector<double> xs = cc::run_iterations(c, iterations, seed0);
  // C_j = X_j / P(colourful) / |Aut|: rescale to the k = kc form cc_median_of_means uses
  std::vector<double> ys(xs);
  if (c->plan.colours() != c->plan.k) {
    long double r = 1;  // [kc^k (kc-k)!/kc!] / [k^k/k!]
    for (int i = 0; i < c->plan.k; ++i)
      r *= ((long double)c->plan.colours() / (c->plan.colours() - i)) / ((long double)c->plan.k / (c->plan.k - i));
    for (auto &y : ys) y = (double)((long double)y * r);
  }
  const cc_status st = cc_median_of_means(ys.data(), iterations, c->plan.k, c->plan.aut, groups, estimate);
  if (st != CC_OK) throw Error(st, "median of means");
  if (per_iter) std::copy(xs.begin(), xs.end(), per_iter);
  API_END(c)
}

cc_status cc_template_info(cc_ctx *c, int64_t *aut, int64_t *aut_root, int32_t *n_steps) {
  API_BEGIN(c)
  if (!c->has_template) throw Error(CC_ERR_STATE, "no template");
  if (aut) *aut = c->plan.aut;
  if (aut_root) *aut_root = c->plan.aut_root;
  if (n_steps) *n_steps = (int32_t)c->plan.steps.size();
  API_END(c)
}

cc_status cc_get_subtree_counts(cc_ctx *c, int32_t x, double *out) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template || !c->has_colors) throw Error(CC_ERR_STATE, "needs graph, template, colouring");
  if (c->pworld() != 1) throw Error(CC_ERR_STATE, "cc_get_subtree_counts needs the whole graph on this rank");
  if (x < 0 || x >= c->plan.k || !out) throw Error(CC_ERR_ARG, "bad template vertex or NULL output");
  // tables are defined for the user's rooting: plan with the fixed root for
  // this call, restore the cost-model plan afterwards
  struct Restore {
    cc_ctx *c;
    ~Restore() {
      try {
        cc::replan(c, false);
      } catch (...) {
      }
    }
  } restore{c};
  cc::replan(c, true);
  const auto &pl = c->plan;
  const auto &R = c->part;
  const int k = pl.colours();
  const int tid = pl.full_table[x];
  std::vector<uint8_t> col((size_t)c->n_crow);
  if (!col.empty()) CUDA_OK(cudaMemcpy(col.data(), c->d_colors, col.size(), cudaMemcpyDeviceToHost));
  double X = 0;
  if (tid == -2) {  // root: per-vertex C(v, T, [k])
    std::memset(out, 0, (size_t)c->n_global * sizeof(double));
    if (pl.k == 1) {
      for (int64_t v = 0; v < c->n_global; ++v) out[v] = 1.0;
    } else {
      std::vector<double> root;
      cc::run_count(c, &X, -1, nullptr, &root);
      for (int64_t i = 0; i < R.n_own; ++i) out[R.own_orig[i]] = root[i];
    }
  } else if (tid == -1) {  // a leaf: the single-vertex table [S == {col v}]
    std::memset(out, 0, (size_t)c->n_global * k * sizeof(double));
    for (int64_t i = 0; i < R.n_own; ++i) out[(size_t)R.own_orig[i] * k + col[i]] = 1.0;
    for (size_t i = 0; i < R.iso_orig.size(); ++i) out[(size_t)R.iso_orig[i] * k + col[c->n_rows + i]] = 1.0;
  } else {  // decompress the table rows into the dense colex layout
    std::vector<double> tab;
    cc::run_count(c, &X, tid, &tab, nullptr);
    const int s = pl.tables[tid].size;
    const int64_t Wd = cc::binom(k, s), Wc = cc::binom(k - 1, s - 1);
    std::memset(out, 0, (size_t)c->n_global * Wd * sizeof(double));
    std::vector<uint32_t> sets((size_t)Wd);
    for (int64_t r = 0; r < Wd; ++r) sets[r] = cc::colex_unrank(s, r);
    const auto &L = c->lay[s];  // storage order of the compressed columns
    for (int64_t i = 0; i < R.n_own; ++i) {
      double *row = out + (size_t)R.own_orig[i] * Wd;
      for (int64_t r = 0; r < Wd; ++r) {
        const int64_t ci = compressed_index(sets[r], col[i]);
        if (ci >= 0) row[r] = tab[(size_t)i * Wc + L.pos[(size_t)ci]];
      }
    }
  }
  API_END(c)
}

cc_status cc_get_subtree_rows(cc_ctx *c, int32_t x, const int32_t *vertices, int32_t nv, double *out) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template || !c->has_colors) throw Error(CC_ERR_STATE, "needs graph, template, colouring");
  if (c->pworld() != 1) throw Error(CC_ERR_STATE, "cc_get_subtree_rows needs the whole graph on this rank");
  if (x < 0 || x >= c->plan.k || nv < 0 || (nv && (!vertices || !out)))
    throw Error(CC_ERR_ARG, "bad template vertex, count or NULL pointer");
  struct Restore {
    cc_ctx *c;
    ~Restore() {
      try {
        cc::replan(c, false);
      } catch (...) {
      }
    }
  } restore{c};
  cc::replan(c, true);
  const auto &pl = c->plan;
  const auto &R = c->part;
  const int k = pl.colours();
  const int tid = pl.full_table[x];
  // original id -> internal row (owned rows only; isolated vertices: -1)
  std::vector<int64_t> inv((size_t)c->n_global, -1);
  for (int64_t i = 0; i < R.n_own; ++i) inv[R.own_orig[i]] = i;
  std::vector<int64_t> rows;
  for (int32_t i = 0; i < nv; ++i) {
    if (vertices[i] < 0 || vertices[i] >= c->n_global) throw Error(CC_ERR_ARG, "vertex id out of range");
    if (inv[vertices[i]] >= 0) rows.push_back(inv[vertices[i]]);
  }
  std::vector<uint8_t> col((size_t)c->n_crow);
  if (!col.empty()) CUDA_OK(cudaMemcpy(col.data(), c->d_colors, col.size(), cudaMemcpyDeviceToHost));
  std::vector<uint8_t> colour_of((size_t)c->n_global, 0);
  for (int64_t i = 0; i < R.n_own; ++i) colour_of[R.own_orig[i]] = col[i];
  for (size_t i = 0; i < R.iso_orig.size(); ++i) colour_of[R.iso_orig[i]] = col[c->n_rows + i];
  double X = 0;
  if (tid == -2) {  // root: per-vertex count, one column
    std::vector<double> root;
    if (pl.k > 1) cc::run_count(c, &X, -1, nullptr, &root);
    for (int32_t i = 0; i < nv; ++i)
      out[i] = pl.k == 1 ? 1.0 : (inv[vertices[i]] >= 0 ? root[inv[vertices[i]]] : 0.0);
  } else if (tid == -1) {  // a leaf: the single-vertex table
    for (int32_t i = 0; i < nv; ++i)
      for (int j = 0; j < k; ++j) out[(size_t)i * k + j] = j == colour_of[vertices[i]] ? 1.0 : 0.0;
  } else {
    std::vector<double> tab;
    if (!rows.empty()) cc::run_count(c, &X, tid, &tab, nullptr, &rows);
    const int s = pl.tables[tid].size;
    const int64_t Wd = cc::binom(k, s), Wc = cc::binom(k - 1, s - 1);
    std::vector<uint32_t> sets((size_t)Wd);
    for (int64_t r = 0; r < Wd; ++r) sets[r] = cc::colex_unrank(s, r);
    size_t j = 0;
    for (int32_t i = 0; i < nv; ++i) {
      double *row = out + (size_t)i * Wd;
      std::fill(row, row + Wd, 0.0);
      if (inv[vertices[i]] < 0) continue;  // isolated: no embedding of a tree with >= 2 vertices
      for (int64_t r = 0; r < Wd; ++r) {
        const int64_t ci = compressed_index(sets[r], colour_of[vertices[i]]);
        if (ci >= 0) row[r] = tab[j * Wc + c->lay[s].pos[(size_t)ci]];
      }
      ++j;
    }
  }
  API_END(c)
}

cc_status cc_set_knob(cc_ctx *c, const char *name, int32_t value) {
  if (!c || !name) return CC_ERR_ARG;
  int *p = knob_ptr(c->knobs, name);
  if (!p) {
    c->err = std::string("unknown knob ") + name;
    return CC_ERR_ARG;
  }
  *p = value;
  ++c->epoch;  // a captured graph no longer matches
  if (std::string(name) == "layout" && c->has_graph && c->has_template) {  // the tables' column order changes
    API_BEGIN(c)
    cc::upload_template(c);
    API_END(c)
  }
  return CC_OK;
}

cc_status cc_get_knob(cc_ctx *c, const char *name, int32_t *value) {
  if (!c || !name || !value) return CC_ERR_ARG;
  int *p = knob_ptr(c->knobs, name);
  if (!p) return CC_ERR_ARG;
  *value = *p;
  return CC_OK;
}

cc_status cc_set_profiling(cc_ctx *c, int32_t on) {
  if (!c) return CC_ERR_ARG;
  c->profiling = on != 0;
  ++c->epoch;
  return CC_OK;
}

cc_status cc_last_profile(cc_ctx *c, double *ms, int32_t cap, int32_t *n) {
  if (!c || !ms) return CC_ERR_ARG;
  const int m = std::min<int>(cap, cc::PH_N + 1);
  for (int i = 0; i < m; ++i) ms[i] = c->prof[i];
  if (m > 1 + cc::PH_COLOR) ms[1 + cc::PH_COLOR] = c->color_ms;
  if (n) *n = m;
  return CC_OK;
}

cc_status cc_last_stats(cc_ctx *c, double *out, int32_t cap) {
  if (!c || !out || cap < 5) return CC_ERR_ARG;
  for (int i = 0; i < std::min<int32_t>(cap, cc::kNStats); ++i) out[i] = c->stats[i];
  return CC_OK;
}

// ---------------------------------------------------------------- host-only
cc_status cc_median_of_means(const double *X, int32_t n, int32_t k, int64_t aut, int32_t groups, double *out) {
  if (!X || !out || n < 1 || groups < 1 || groups > n || k < 1 || aut < 1) return CC_ERR_ARG;
  long double scale = 1;  // k^k / k!
  for (int i = 1; i <= k; ++i) scale *= (long double)k / i;
  std::vector<long double> z((size_t)groups);
  int64_t pos = 0;
  for (int g = 0; g < groups; ++g) {  // equal sizes in iteration order, remainder from the front
    const int64_t size = n / groups + (g < n % groups ? 1 : 0);
    long double s = 0;
    for (int64_t j = 0; j < size; ++j) s += (long double)X[pos + j];
    pos += size;
    z[g] = s / size * scale / (long double)aut;
  }
  std::sort(z.begin(), z.end());
  *out = (double)(groups % 2 ? z[groups / 2] : (z[groups / 2 - 1] + z[groups / 2]) / 2);
  return CC_OK;
}

cc_status cc_niter(double eps, double delta, int32_t k, double constant, int64_t *out) {
  if (!out || !(eps > 0) || !(delta > 0) || !(delta <= 1) || k < 1 || !(constant > 0)) return CC_ERR_ARG;
  const double v = std::ceil(constant * std::exp((double)k) * std::log(1.0 / delta) / (eps * eps));
  *out = v < 1 ? 1 : (int64_t)v;
  return CC_OK;
}

int64_t cc_colex_rank(uint32_t mask) { return mask >> cc::kMaxK ? -1 : cc::colex_rank(mask); }

uint32_t cc_colex_unrank(int32_t s, int64_t r) {
  if (s < 0 || s > cc::kMaxK || r < 0 || r >= cc::binom(cc::kMaxK, s)) return 0xFFFFFFFFu;
  return cc::colex_unrank(s, r);
}

cc_status cc_split_table(int32_t k, int32_t t, int32_t a, uint32_t *out, int64_t cap) {
  if (k < 1 || k > cc::kMaxK || t < 2 || t > k || a < 1 || a >= t || !out) return CC_ERR_ARG;
  auto tab = cc::split_table(k, t, a);
  if ((int64_t)tab.size() > cap) return CC_ERR_ARG;
  std::copy(tab.begin(), tab.end(), out);
  return CC_OK;
}

cc_status cc_zblock_table(int32_t K, int32_t ts, int32_t as, uint16_t *out, int64_t cap, int32_t *n_blocks,
                          int32_t *ld) {
  if (K < 2 || K > cc::kMaxK || ts < 2 || ts >= K || as < 1 || as >= ts || !n_blocks || !ld) return CC_ERR_ARG;
  int nb = 0;
  auto tab = cc::zblock_table(K, ts, as, &nb);
  *n_blocks = nb;
  *ld = (int32_t)cc::zblock_ld(ts, as);
  if (out) {
    if ((int64_t)tab.size() > cap) return CC_ERR_ARG;
    std::copy(tab.begin(), tab.end(), out);
  }
  return CC_OK;
}

cc_status cc_plan_template(int32_t k, const int32_t *parent, int32_t *steps_out, int32_t cap_steps, int32_t *n_steps,
                           int64_t *aut, int64_t *aut_root, double *memory, double *computation) {
  try {
    cc::Plan p = cc::make_plan(k, parent);
    if (n_steps) *n_steps = (int32_t)p.steps.size();
    if (steps_out) {
      if (cap_steps < (int32_t)p.steps.size()) return CC_ERR_ARG;
      for (size_t s = 0; s < p.steps.size(); ++s) {
        const auto &st = p.steps[s];
        int32_t *o = steps_out + 6 * s;
        o[0] = st.t;
        o[1] = st.a;
        o[2] = st.p;
        o[3] = st.active;
        o[4] = st.passive;
        o[5] = st.out;
      }
    }
    if (aut) *aut = p.aut;
    if (aut_root) *aut_root = p.aut_root;
    if (memory) *memory = p.memory;
    if (computation) *computation = p.computation;
  } catch (const Error &e) {
    return e.status;
  }
  return CC_OK;
}

cc_status cc_plan_template_auto(int32_t k, const int32_t *parent, double avg_degree, int32_t elem,
                                int32_t *steps_out, int32_t cap_steps, int32_t *n_steps, int32_t *root,
                                double *cost) {
  try {
    if (elem != 4 && elem != 8) return CC_ERR_ARG;
    cc::PlanOpts o;
    o.auto_root = true;
    o.avg_degree = avg_degree;
    o.elem = elem;
    cc::Plan p = cc::make_plan(k, parent, &o);
    if (n_steps) *n_steps = (int32_t)p.steps.size();
    if (steps_out) {
      if (cap_steps < (int32_t)p.steps.size()) return CC_ERR_ARG;
      for (size_t s = 0; s < p.steps.size(); ++s) {
        const auto &st = p.steps[s];
        int32_t *out = steps_out + 6 * s;
        out[0] = st.t;
        out[1] = st.a;
        out[2] = st.p;
        out[3] = st.active;
        out[4] = st.passive;
        out[5] = st.out;
      }
    }
    if (root) *root = p.root;
    if (cost) *cost = cc::plan_cost(p, o);
  } catch (const Error &e) {
    return e.status;
  }
  return CC_OK;
}

cc_status cc_partition_plan(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t world, int32_t rank,
                            uint64_t relabel_seed, int64_t *sizes_out, int32_t *own_orig, int32_t *halo_orig,
                            int64_t *recv_off, int64_t *send_off, int32_t *send_idx, int64_t *rp, int32_t *lcol) {
  try {
    if (!sizes_out) return CC_ERR_ARG;
    cc::HostGraph g = cc::validate_graph(n, row_ptr, col);
    cc::RankPart R = cc::partition_graph(g, world, rank, relabel_seed);
    sizes_out[0] = R.n_own;
    sizes_out[1] = R.n_halo;
    sizes_out[2] = (int64_t)R.col.size();
    sizes_out[3] = R.send_off.back();
    if (own_orig) std::copy(R.own_orig.begin(), R.own_orig.end(), own_orig);
    if (halo_orig) std::copy(R.halo_orig.begin(), R.halo_orig.end(), halo_orig);
    if (recv_off) std::copy(R.recv_off.begin(), R.recv_off.end(), recv_off);
    if (send_off) std::copy(R.send_off.begin(), R.send_off.end(), send_off);
    if (send_idx) std::copy(R.send_idx.begin(), R.send_idx.end(), send_idx);
    if (rp) std::copy(R.rp.begin(), R.rp.end(), rp);
    if (lcol) std::copy(R.col.begin(), R.col.end(), lcol);
  } catch (const Error &e) {
    return e.status;
  }
  return CC_OK;
}

cc_status cc_exchange_model(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t world, int32_t rank,
                            uint64_t relabel_seed, double row_bytes, double *out) {
  try {
    if (!out || world < 2 || rank < 0 || rank >= world || !(row_bytes > 0)) return CC_ERR_ARG;
    cc::HostGraph g = cc::validate_graph(n, row_ptr, col);
    cc::RankPart R = cc::partition_graph(g, world, rank, relabel_seed);
    const cc::ExchangeModel m = cc::model_exchange(R, cc::peer_bounds(R), row_bytes);
    out[0] = m.grouped_s;
    out[1] = m.ring_s;
    out[2] = m.link_bps;
    out[3] = m.gather_bps;
  } catch (const Error &e) {
    return e.status;
  }
  return CC_OK;
}

}  // extern "C"
