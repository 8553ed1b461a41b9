// ctx.h -- the library context (one per rank) and the executor interface.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "loopback.h"
#include "nccl_dl.h"

#define CUDA_OK(expr)                                                                                  \
  do {                                                                                                 \
    cudaError_t e_ = (expr);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      throw cc::Error(e_ == cudaErrorMemoryAllocation ? CC_ERR_OOM : CC_ERR_CUDA,                      \
                      std::string(#expr) + ": " + cudaGetErrorString(e_));                             \
  } while (0)

#define NCCL_OK(expr)                                                                                  \
  do {                                                                                                 \
    ncclResult_t r_ = (expr);                                                                          \
    if (r_ != ncclSuccess)                                                                             \
      throw cc::Error(CC_ERR_NCCL, std::string(#expr) + ": " + cc::nccl().GetErrorString(r_));        \
  } while (0)

namespace cc {

struct DevX;  // device-initiated exchange state (devx.cu)

constexpr int kNStats = 16;  // cc_last_stats entries

// Phases reported by cc_last_profile after "total": PROFILE order.
enum Phase { PH_COLOR = 0, PH_CSORT, PH_HIST, PH_GATHER, PH_COMBINE, PH_ROOT, PH_EXCHANGE, PH_EXPOSED, PH_N };

// One aggregation pass over a range [beg[v], end[v]) of every owned row.
struct Pass {
  int32_t *light = nullptr;
  int32_t *seg_v = nullptr, *seg_hv = nullptr, *hv_first = nullptr, *hv_nseg = nullptr;
  int64_t *seg_b = nullptr, *seg_e = nullptr;
  int64_t n_light = 0, n_seg = 0, n_hv = 0;
  int64_t small_from = 0;      // first item (segments first, then light) of the <= 8-neighbour tail
  int64_t split[8] = {0};      // split[i]: first item of the <= (8 << i)-neighbour tail
  int64_t seg_len = 0;         // segment length s of the heavy items
  int64_t nnz = 0;             // adjacency entries covered
  std::vector<int64_t> pref;   // host: adjacency entries before item i (items() + 1 entries)
  std::vector<int32_t> light_h;  // host copy of the light items' vertices (increasing)
  int64_t max_heavy_v = -1;      // largest vertex with heavy segments
  const int64_t *beg = nullptr, *end = nullptr;  // device
  uint16_t *goff = nullptr;    // n_items x 16 colour-group ends (per colouring)
  dev::ItemDesc *desc = nullptr;  // n_items descriptors (per colouring)
  int32_t *col_sorted = nullptr;   // the colour-sorted neighbour ids this pass reads
  int64_t items() const { return n_seg + n_light; }
  dev::AggWork view() const {
    dev::AggWork w;
    w.light = light;
    w.n_light = n_light;
    w.seg_v = seg_v;
    w.seg_b = seg_b;
    w.seg_e = seg_e;
    w.seg_hv = seg_hv;
    w.hv_first = hv_first;
    w.hv_nseg = hv_nseg;
    w.n_seg = n_seg;
    w.n_hv = n_hv;
    return w;
  }
};

// A stream-ordered device buffer shared by several table handles (a lift
// step's table is the very buffer of its neighbour sum).
struct Buf {
  void *p = nullptr;
  size_t bytes = 0;
  int refs = 0;
  bool owned = true;  // false: owned by a TableCache (never freed by the executor)
};

// Tables of one colouring shared across the templates of
// cc_count_colorful_multi: isomorphic rooted sub-templates
// (same AHU code, Plan::tables[].code) have identical tables for the same
// colouring and colour universe, so each is computed once.  The colour sort
// and the leaf level are computed once as well.
struct TableCache {
  std::map<std::string, std::pair<void *, size_t>> tables;  // code -> device buffer, bytes
  void *hist = nullptr;
  size_t hist_bytes = 0;
  bool sorted = false;
  size_t bytes = 0, budget = 0;
  int64_t reused = 0, stored = 0;
};

}  // namespace cc

struct cc_ctx {
  cc_options opt{};
  cc::dev::Knobs knobs;  // implementation switches (env at cc_create, cc_set_knob)
  std::string err;
  bool poisoned = false;
  int num_sms = 148;
  double total_mem = 0;  // device memory (bytes), at cc_create
  int64_t l2_bytes = 126LL << 20;
  cudaStream_t s_main = nullptr, s_comm = nullptr;
  ncclComm_t comm = nullptr;
  cc::LoopbackGroup *loop = nullptr;  // in-process transport instead of NCCL (test hook)
  std::vector<void *> persistent;  // cudaMalloc'd: graph, plan tables (freed on reload / destroy)

  // graph
  bool has_graph = false;
  cc::RankPart part;
  int64_t n_global = 0, n_own = 0, n_halo = 0, n_rows = 0;
  int64_t n_crow = 0;  // coloured rows: owned | halo | isolated
  int64_t *d_rp = nullptr, *d_mid = nullptr;
  int32_t *d_col = nullptr, *d_col_sorted = nullptr, *d_orig = nullptr, *d_send_idx = nullptr;
  uint8_t *d_colors = nullptr;
  uint8_t *d_color_stage = nullptr;  // n_global bytes: a caller's colouring in original order
  unsigned *d_bad = nullptr;
  cc::Pass p_full, p_local, p_remote;  // world 1: p_full; world > 1: p_local + p_remote (+ p_full for hist)
  std::vector<cc::Pass> p_peer;        // ring exchange: the remote pass per source peer (replaces p_remote)
  int xmode = 0;                       // exchange schedule in use: 0 none, CC_EXCHANGE_GROUPED / _RING / ...
  int64_t a2a_rows = 0;
  int64_t max_halo = 0;                // halo rows of the largest rank (window size)                // CC_EXCHANGE_ALLTOALL: rows per peer block (max over all rank pairs)
  cc::DevX *devx = nullptr;            // CC_EXCHANGE_DEVICE: device communicator + halo window
  // column chunks: chunk_cols > 0 splits every neighbour sum's
  // passive columns into launches of that width; chunked (world > 1) then
  // exchanges halo rows per chunk into double buffers and tables keep only
  // the owned rows
  int64_t chunk_cols = 0;
  bool chunked = false;
  double xmodel[2] = {0, 0};           // modelled grouped / ring seconds (max over ranks)
  int64_t max_seg = 0, max_hv = 0;
  // adjacency entries per non-isolated vertex of the GLOBAL graph: the
  // planner's statistic, identical on every rank (a per-rank figure could
  // pick different plans on different ranks, and their exchanges would not match)
  double avg_degree = 0;
  // CUDA graph of a count (use_graphs): rebuilt when epoch moves past gepoch
  int64_t epoch = 0, gepoch = -1;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t graph_ev[2] = {nullptr, nullptr};

  // template
  bool has_template = false;
  std::vector<int32_t> user_parent;  // the template as given (re-planned when the graph changes)
  int user_kc = 0;                   // colours of the colouring (0 = template size)
  cc::Plan plan;
  std::vector<uint32_t *> d_split;    // per step: split table (combine steps)
  std::vector<uint16_t *> d_ztab;     // per step: Z-block cover table (nullptr if none)
  std::vector<int> zblocks;
  std::vector<uint16_t *> d_map;      // per passive size p: gather map (p >= 2)
  std::vector<uint32_t *> d_skip;     // per passive size p: sector-skip table
  std::vector<int> skip_words;
  std::vector<cc::Layout> lay;        // per table size t: storage order of the C(k-1, t-1) columns (R-3)
  uint16_t *d_comp = nullptr;         // root step complement table
  bool has_colors = false;
  bool sorted_valid = false;          // colour-sorted adjacency matches the colouring
  bool full_sorted_valid = false;     // world > 1: the full ranges' sort (fused root) matches it
  int32_t *d_col_sorted_full = nullptr;

  // scratch
  double *d_partials = nullptr, *d_result = nullptr;
  int n_partials = 0;
  unsigned int *d_arrive = nullptr;
  int64_t arrive_cap = 0;

  // profile / stats of the last count
  double prof[cc::PH_N + 1] = {0};
  double stats[cc::kNStats] = {0};
  std::vector<std::pair<size_t, double>> gather_log;  // (ev_log index, algorithmic bytes) per gather launch
  int gather_ordinal = 0;                             // neighbour-sum passes launched in this count
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_log;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t ev_color[2] = {nullptr, nullptr};
  double color_ms = 0;
  size_t cur_bytes = 0, peak_bytes = 0;

  int elem() const { return opt.precision == CC_FP64 ? 8 : 4; }
  // ranks of the 1D vertex partition (1 in replica mode: each rank has the whole graph)
  int pworld() const { return opt.replicas ? 1 : opt.world; }
  int64_t ld_of(int64_t W) const {
    const int64_t m = 32 / elem();
    return (std::max<int64_t>(W, 1) + m - 1) / m * m;
  }

  template <typename T>
  T *pmalloc(size_t count) {
    T *d = nullptr;
    if (!count) return nullptr;
    CUDA_OK(cudaMalloc(&d, count * sizeof(T)));
    persistent.push_back(d);
    return d;
  }
  template <typename T>
  T *pupload(const std::vector<T> &h) {
    T *d = pmalloc<T>(h.size());
    if (d) CUDA_OK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  void pfree(void *p) {
    if (!p) return;
    auto it = std::find(persistent.begin(), persistent.end(), p);
    if (it != persistent.end()) persistent.erase(it);
    cudaFree(p);
  }
  void *amalloc(size_t bytes, cudaStream_t s) {
    void *p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(bytes, 256), s);
    if (e == cudaErrorMemoryAllocation) {
      // freed blocks stay mapped in the pool (release threshold = max) and may
      // be too fragmented for one large table: return them and retry once
      (void)cudaGetLastError();
      cudaMemPool_t pool;
      CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, opt.device));
      CUDA_OK(cudaStreamSynchronize(s));
      CUDA_OK(cudaMemPoolTrimTo(pool, 0));
      e = cudaMallocAsync(&p, std::max<size_t>(bytes, 256), s);
    }
    CUDA_OK(e);
    cur_bytes += bytes;
    peak_bytes = std::max(peak_bytes, cur_bytes);
    return p;
  }
  void afree(void *&p, size_t bytes, cudaStream_t s) {
    if (!p) return;
    CUDA_OK(cudaFreeAsync(p, s));
    cur_bytes -= bytes;
    p = nullptr;
  }
  cudaEvent_t ev() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  bool profiling = true;     // cc_set_profiling
  bool phase_events = true;  // per-kernel event pairs for cc_last_profile (knob phase_events = 0: off)
  // SMs the gathers may fill: all, or all but knobs.grid_reserve while a halo
  // exchange over NCCL is in flight (NCCL's kernels need SMs to progress)
  int gather_sms(bool exchanging) const {
    const int r = knobs.grid_reserve >= 0 ? knobs.grid_reserve : (exchanging && comm ? 8 : 0);
    return exchanging ? std::max(1, num_sms - r) : num_sms;
  }
  cudaEvent_t begin(cudaStream_t s) {
    if (!phase_events) return nullptr;
    cudaEvent_t b = ev();
    CUDA_OK(cudaEventRecord(b, s));
    return b;
  }
  void end(int ph, cudaStream_t s, cudaEvent_t b) {
    if (!phase_events || !b) return;
    cudaEvent_t e = ev();
    CUDA_OK(cudaEventRecord(e, s));
    ev_log.push_back({ph, {b, e}});
  }
  void check_launch() { CUDA_OK(cudaGetLastError()); }
};

namespace cc {
// exec.cu
void load_graph(cc_ctx *c, const HostGraph &g);
void upload_template(cc_ctx *c);
// (Re)plan c->user_parent: fixed root if `fixed` or opt.fixed_root, else the
// cost-model root for the loaded graph's average degree and table precision.
void replan(cc_ctx *c, bool fixed);
void launch_colouring(cc_ctx *c, uint64_t seed);
// One colouring's DP.  dump_table >= 0 keeps every table and returns table
// `dump_table` (compressed rows, owned order) in *dump; root_out receives the
// per-vertex root values.
// dump_table >= 0: copy that table (compressed rows) into *dump -- every
// owned row (dump_rows == nullptr; disables the fused root and releases) or
// only the internal rows listed in *dump_rows (copied right after the step
// that produces the table; nothing else changes).
// capture: record the device work into the stream's capture (CUDA graph), no host copies
void run_count(cc_ctx *c, double *X, int dump_table, std::vector<double> *dump, std::vector<double> *root_out,
               const std::vector<int64_t> *dump_rows = nullptr, TableCache *cache = nullptr, bool capture = false);
// cc_count_colorful through a captured CUDA graph (use_graphs, one rank)
void count_graph(cc_ctx *c, double *X);
// devx.cu: the device-initiated exchange (CC_EXCHANGE_DEVICE)
void devx_init(cc_ctx *c, const std::vector<int64_t> &dst_row);
void devx_free(cc_ctx *c);
void *devx_window(cc_ctx *c, size_t bytes);
void devx_put(cc_ctx *c, const void *P, int64_t ldP, int64_t c0, int64_t w, size_t win_off, int64_t ldH);
cc_status device_selftest(int32_t device);
void free_cache(cc_ctx *c, TableCache &cache);
// X_j for colourings seed0 + j, j < iterations (replica mode with world > 1:
// iteration j on rank j mod world, then one all-reduce of the vector).
std::vector<double> run_iterations(cc_ctx *c, int iterations, uint64_t seed0);
}  // namespace cc
