// ctx.cu -- the context, the per-colouring step executor and the C ABI.
//
// One cc_count_colorful = PAPER.md Alg. 1 lines 8-10 (Eq. 2) for one
// colouring, distributed as Alg. 2 (lines 199-243) when world > 1:
//   for each step (t; a, p) of the plan (sub-templates in reverse partition
//   order):
//     N <- neighbour sum of the passive table (once per distinct passive);
//          world > 1: the passive table's boundary rows are exchanged with
//          grouped NCCL send/recv on a comm stream while the local part of
//          the neighbour sum runs (pipelining);
//     T <- split-sum combine of the active table with N (or a lift, a = 1);
//   X = sum_v of the root step (fp64), all-reduced over ranks (line 237).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.h"
#include "kernels.cuh"
#include "nccl_dl.h"

using cc::Error;

#define CUDA_OK(expr)                                                                                  \
  do {                                                                                                 \
    cudaError_t e_ = (expr);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      throw Error(e_ == cudaErrorMemoryAllocation ? CC_ERR_OOM : CC_ERR_CUDA,                          \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                                 \
  } while (0)

#define NCCL_OK(expr)                                                                                  \
  do {                                                                                                 \
    ncclResult_t r_ = (expr);                                                                          \
    if (r_ != ncclSuccess) throw Error(CC_ERR_NCCL, std::string(#expr) + ": " + cc::nccl().GetErrorString(r_)); \
  } while (0)

namespace {

enum Phase { PH_COLOR = 0, PH_HIST, PH_AGG, PH_LIFT, PH_COMBINE, PH_ROOT, PH_EXCHANGE, PH_N };

struct WorkDev {
  int32_t *light = nullptr;
  int32_t *seg_v = nullptr, *seg_hv = nullptr, *hv_first = nullptr, *hv_nseg = nullptr;
  int64_t *seg_b = nullptr, *seg_e = nullptr;
  int64_t n_light = 0, n_seg = 0, n_hv = 0;
  int64_t nnz = 0;  // adjacency entries covered by this pass
  cc::dev::AggWork view() const {
    cc::dev::AggWork w;
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

template <typename T>
T *dmalloc_copy(const std::vector<T> &h) {
  T *d = nullptr;
  if (h.empty()) return nullptr;
  CUDA_OK(cudaMalloc(&d, h.size() * sizeof(T)));
  CUDA_OK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

struct cc_ctx {
  cc_options opt{};
  std::string err;
  bool poisoned = false;
  int num_sms = 148;
  cudaStream_t s_main = nullptr, s_comm = nullptr;
  ncclComm_t comm = nullptr;
  std::vector<void *> persistent;  // cudaMalloc'd, freed in destroy

  // graph
  bool has_graph = false;
  cc::RankPart part;
  int64_t n_global = 0, n_own = 0, n_halo = 0, n_rows = 0;
  int64_t n_crow = 0;  // coloured rows: owned | halo | isolated
  int64_t *d_rp = nullptr, *d_mid = nullptr;
  int32_t *d_col = nullptr, *d_orig = nullptr, *d_send_idx = nullptr;
  uint8_t *d_colors = nullptr;
  WorkDev w_full, w_local, w_remote;
  int64_t max_hv = 0, max_seg = 0;

  // template
  bool has_template = false;
  cc::Plan plan;
  std::vector<uint32_t *> d_split;  // per step (combine steps)
  std::vector<uint16_t *> d_drop;   // per step (lift steps)
  uint16_t *d_comp = nullptr;       // root step complement table
  bool has_colors = false;

  // scratch
  double *d_partials = nullptr, *d_result = nullptr;
  int n_partials = 0;
  unsigned int *d_arrive = nullptr;
  int64_t arrive_cap = 0;

  // profile / stats of the last count
  double prof[PH_N + 1] = {0};
  double stats[5] = {0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_log;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  bool profile = true;
  size_t cur_bytes = 0, peak_bytes = 0;
  cudaEvent_t ev_color[2] = {nullptr, nullptr};
  double color_ms = 0;

  int elem() const { return opt.precision == CC_FP64 ? 8 : 4; }
  int64_t ld_of(int W) const { return round_up(std::max(W, 1), 32 / elem()); }

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
  void pfree(void *&p) {
    if (!p) return;
    auto it = std::find(persistent.begin(), persistent.end(), p);
    if (it != persistent.end()) persistent.erase(it);
    cudaFree(p);
    p = nullptr;
  }
  void *amalloc(size_t bytes, cudaStream_t s) {
    void *p = nullptr;
    CUDA_OK(cudaMallocAsync(&p, std::max<size_t>(bytes, 256), s));
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
  void begin(int ph, cudaStream_t s, cudaEvent_t *b) {
    if (!profile) return;
    *b = ev();
    CUDA_OK(cudaEventRecord(*b, s));
    (void)ph;
  }
  void end(int ph, cudaStream_t s, cudaEvent_t b) {
    if (!profile) return;
    cudaEvent_t e = ev();
    CUDA_OK(cudaEventRecord(e, s));
    ev_log.push_back({ph, {b, e}});
  }
  void check_launch() { CUDA_OK(cudaGetLastError()); }
};

namespace {

// ---------------------------------------------------------------- work lists
void build_work(cc_ctx *c, const std::vector<int64_t> &beg, const std::vector<int64_t> &end, bool skip_empty,
                WorkDev &w) {
  const int64_t L = c->opt.segment_len > 0 ? c->opt.segment_len : 4096;
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
  w.n_seg = (int64_t)seg_v.size();
  w.n_hv = (int64_t)hv_first.size();
  w.light = c->pupload(light);
  w.seg_v = c->pupload(seg_v);
  w.seg_hv = c->pupload(seg_hv);
  w.hv_first = c->pupload(hv_first);
  w.hv_nseg = c->pupload(hv_nseg);
  w.seg_b = c->pupload(seg_b);
  w.seg_e = c->pupload(seg_e);
  c->max_hv = std::max(c->max_hv, w.n_hv);
  c->max_seg = std::max(c->max_seg, w.n_seg);
}

void free_graph(cc_ctx *c) {
  for (void *p : c->persistent) cudaFree(p);
  c->persistent.clear();
  c->d_rp = c->d_mid = nullptr;
  c->d_col = c->d_orig = c->d_send_idx = nullptr;
  c->d_colors = nullptr;
  c->w_full = c->w_local = c->w_remote = WorkDev();
  c->d_split.clear();
  c->d_drop.clear();
  c->d_comp = nullptr;
  c->d_partials = c->d_result = nullptr;
  c->d_arrive = nullptr;
  c->arrive_cap = 0;
  c->max_hv = c->max_seg = 0;
  c->has_graph = c->has_template = c->has_colors = false;
}

void upload_template(cc_ctx *c) {
  using namespace cc;
  for (auto *p : c->d_split) { void *q = p; c->pfree(q); }
  for (auto *p : c->d_drop) { void *q = p; c->pfree(q); }
  if (c->d_comp) { void *q = c->d_comp; c->pfree(q); }
  c->d_split.assign(c->plan.steps.size(), nullptr);
  c->d_drop.assign(c->plan.steps.size(), nullptr);
  c->d_comp = nullptr;
  const int k = c->plan.k;
  for (size_t s = 0; s < c->plan.steps.size(); ++s) {
    const Step &st = c->plan.steps[s];
    if (st.out < 0) c->d_comp = c->pupload(complement_table(k, st.a));
    else if (st.a == 1) c->d_drop[s] = c->pupload(drop_table(k, st.t));
    else c->d_split[s] = c->pupload(split_table(k, st.t, st.a));
  }
}

// ---------------------------------------------------------------- aggregation
// N = sum over neighbours of the passive table P (rows n_own[+halo] x ldP).
void aggregate(cc_ctx *c, void *P, int W, void *N) {
  using namespace cc::dev;
  const int elem = c->elem();
  const int64_t ld = c->ld_of(W);
  const int nch = agg_nchunks(elem, W, c->opt.chunk_cols);
  auto run_pass = [&](const WorkDev &w, const int64_t *beg, const int64_t *end, int accumulate) {
    AggArgs a;
    a.beg = beg;
    a.end = end;
    a.col = c->d_col;
    a.src = P;
    a.ld_src = ld;
    a.dst = N;
    a.ld_dst = ld;
    a.W = W;
    a.accumulate = accumulate;
    a.work = w.view();
    a.ld_scratch = round_up(W, 4);
    void *scratch = nullptr;
    size_t sbytes = (size_t)w.n_seg * a.ld_scratch * sizeof(double);
    if (w.n_seg) {
      scratch = c->amalloc(sbytes, c->s_main);
      const int64_t need = w.n_hv * nch;
      if (need > c->arrive_cap) {
        void *q = c->d_arrive;
        c->pfree(q);
        c->d_arrive = c->pmalloc<unsigned int>((size_t)need);
        c->arrive_cap = need;
      }
      CUDA_OK(cudaMemsetAsync(c->d_arrive, 0, (size_t)need * sizeof(unsigned int), c->s_main));
    }
    a.scratch = static_cast<double *>(scratch);
    a.arrive = c->d_arrive;
    cudaEvent_t b;
    c->begin(PH_AGG, c->s_main, &b);
    c->stats[3] += launch_agg(elem, a, c->opt.chunk_cols, c->num_sms, nullptr, c->s_main);
    c->check_launch();
    c->end(PH_AGG, c->s_main, b);
    if (scratch) c->afree(scratch, sbytes, c->s_main);
    // model bytes: index stream + gathered rows + rows written (+ read when accumulating)
    const double bytes = (double)w.nnz * (4.0 + (double)W * elem) +
                         (double)(w.n_light + w.n_hv) * W * elem * (1 + accumulate);
    c->stats[0] += (double)w.nnz * W;
    c->stats[1] += bytes;
    c->stats[2] += bytes;
  };
  if (c->opt.world == 1) {
    run_pass(c->w_full, c->d_rp, c->d_rp + 1, 0);
    return;
  }
  // world > 1: exchange the boundary rows of P on the comm stream while the
  // local part runs; then add the remote part.
  auto &api = cc::nccl();
  cudaEvent_t ready = c->ev(), recvd = c->ev();
  CUDA_OK(cudaEventRecord(ready, c->s_main));
  CUDA_OK(cudaStreamWaitEvent(c->s_comm, ready, 0));
  const auto &R = c->part;
  const int64_t send_rows = R.send_off[c->opt.world];
  const size_t sbytes = (size_t)send_rows * ld * elem;
  void *sendbuf = send_rows ? c->amalloc(sbytes, c->s_comm) : nullptr;
  cudaEvent_t xb;
  c->begin(PH_EXCHANGE, c->s_comm, &xb);
  c->stats[3] += launch_pack(elem, P, ld, c->d_send_idx, send_rows, sendbuf, c->s_comm);
  c->check_launch();
  const ncclDataType_t dt = elem == 8 ? ncclFloat64 : ncclFloat32;
  NCCL_OK(api.GroupStart());
  for (int q = 0; q < c->opt.world; ++q) {
    if (q == c->opt.rank) continue;
    const int64_t ns = R.send_off[q + 1] - R.send_off[q];
    const int64_t nr = R.recv_off[q + 1] - R.recv_off[q];
    if (ns) NCCL_OK(api.Send(static_cast<char *>(sendbuf) + (size_t)R.send_off[q] * ld * elem, (size_t)(ns * ld),
                             dt, q, c->comm, c->s_comm));
    if (nr) NCCL_OK(api.Recv(static_cast<char *>(P) + (size_t)(c->n_own + R.recv_off[q]) * ld * elem,
                             (size_t)(nr * ld), dt, q, c->comm, c->s_comm));
  }
  NCCL_OK(api.GroupEnd());
  c->end(PH_EXCHANGE, c->s_comm, xb);
  if (sendbuf) c->afree(sendbuf, sbytes, c->s_comm);
  CUDA_OK(cudaEventRecord(recvd, c->s_comm));
  run_pass(c->w_local, c->d_rp, c->d_mid, 0);
  CUDA_OK(cudaStreamWaitEvent(c->s_main, recvd, 0));
  run_pass(c->w_remote, c->d_mid, c->d_rp + 1, 1);
  c->stats[1] += (double)send_rows * ld * elem * 2;
}

// ---------------------------------------------------------------- one colouring
// keep_all: keep every table (for cc_get_subtree_counts); dump_table / per_vertex
// receive the requested table id (device copy to host) / root per-vertex values.
void run_count(cc_ctx *c, double *X, int dump_table, std::vector<double> *dump_out, std::vector<double> *root_out) {
  using namespace cc;
  using namespace cc::dev;
  const Plan &pl = c->plan;
  const int k = pl.k, elem = c->elem();
  std::fill(c->stats, c->stats + 5, 0.0);
  c->ev_used = 0;
  c->ev_log.clear();
  c->cur_bytes = c->peak_bytes = 0;
  if (k == 1) {  // the single-vertex template maps onto every vertex
    *X = (double)c->n_global;
    std::fill(c->prof, c->prof + PH_N + 1, 0.0);
    return;
  }
  const int64_t n = c->n_own, rows = c->n_rows;
  cudaEvent_t t0 = c->ev(), t1 = c->ev();
  CUDA_OK(cudaEventRecord(t0, c->s_main));
  const int nt = (int)pl.tables.size();
  std::vector<void *> T(nt, nullptr), Nb(nt, nullptr);
  std::vector<size_t> Tbytes(nt, 0), Nbytes(nt, 0);
  void *hist = nullptr;
  size_t hist_bytes = 0;
  double *per_vertex = nullptr;
  if (root_out) per_vertex = static_cast<double *>(c->amalloc((size_t)std::max<int64_t>(n, 1) * 8, c->s_main));

  for (int s = 0; s < (int)pl.steps.size(); ++s) {
    const Step &st = pl.steps[s];
    const int Wt = (int)binom(k, st.t), Wa = (int)binom(k, st.a), Wp = (int)binom(k, st.p);
    const void *Np;
    int64_t ldN;
    if (st.p == 1) {
      if (!hist) {
        hist_bytes = (size_t)n * c->ld_of(k) * elem;
        hist = c->amalloc(hist_bytes, c->s_main);
        cudaEvent_t b;
        c->begin(PH_HIST, c->s_main, &b);
        c->stats[3] += launch_hist(elem, c->d_rp, c->d_rp + 1, c->d_col, c->d_colors, c->w_full.view(), n, k, hist,
                                   c->ld_of(k), c->num_sms, c->s_main);
        c->check_launch();
        c->end(PH_HIST, c->s_main, b);
        const double nnz = (double)c->part.col.size();
        c->stats[0] += nnz * k;  // U counts C(k,1) = k colour sets per adjacency entry
        c->stats[1] += nnz * 5.0 + (double)n * k * elem;
      }
      Np = hist;
      ldN = c->ld_of(k);
    } else {
      const int P = st.passive;
      if (!Nb[P]) {
        Nbytes[P] = (size_t)n * c->ld_of(Wp) * elem;
        Nb[P] = c->amalloc(Nbytes[P], c->s_main);
        aggregate(c, T[P], Wp, Nb[P]);
      }
      Np = Nb[P];
      ldN = c->ld_of(Wp);
    }
    if (st.out < 0) {  // root step fused with the sum over v (Eq. 3)
      cudaEvent_t b;
      c->begin(PH_ROOT, c->s_main, &b);
      const void *A = st.active >= 0 ? T[st.active] : nullptr;
      c->stats[3] += launch_root(elem, A, c->ld_of(Wa), Wa, Np, ldN, c->d_comp, c->d_colors, n, c->d_partials,
                                 c->n_partials, per_vertex, c->d_result, c->s_main);
      c->check_launch();
      c->end(PH_ROOT, c->s_main, b);
      c->stats[1] += (double)n * (st.active >= 0 ? 2.0 * Wa : 1.0) * elem;
    } else {
      Tbytes[st.out] = (size_t)rows * c->ld_of(Wt) * elem;
      T[st.out] = c->amalloc(Tbytes[st.out], c->s_main);
      cudaEvent_t b;
      if (st.a == 1) {
        c->begin(PH_LIFT, c->s_main, &b);
        c->stats[3] += launch_lift(elem, Np, ldN, c->d_colors, c->d_drop[s], n, Wt, T[st.out], c->ld_of(Wt),
                                   c->num_sms, c->s_main);
        c->check_launch();
        c->end(PH_LIFT, c->s_main, b);
        c->stats[1] += (double)n * (Wt + (double)binom(k - 1, st.t - 1)) * elem;
      } else {
        c->begin(PH_COMBINE, c->s_main, &b);
        c->stats[3] += launch_combine(elem, T[st.active], c->ld_of(Wa), Wa, Np, ldN, st.p == 1 ? k : Wp, c->d_split[s],
                                      (int)binom(st.t, st.a), n, T[st.out], c->ld_of(Wt), Wt, c->num_sms,
                                      c->s_main);
        c->check_launch();
        c->end(PH_COMBINE, c->s_main, b);
        c->stats[1] += (double)n * (Wa + Wp + Wt) * elem;
      }
    }
    if (dump_table < 0) {  // free dead tables / neighbour sums
      for (int id = 0; id < nt; ++id) {
        if (T[id] && pl.table_last_use[id] == s) c->afree(T[id], Tbytes[id], c->s_main);
        if (Nb[id] && pl.n_last_use[id] == s) c->afree(Nb[id], Nbytes[id], c->s_main);
      }
    }
  }
  if (c->opt.world > 1) {
    cudaEvent_t b;
    c->begin(PH_EXCHANGE, c->s_main, &b);
    NCCL_OK(cc::nccl().AllReduce(c->d_result, c->d_result, 1, ncclFloat64, ncclSum, c->comm, c->s_main));
    c->end(PH_EXCHANGE, c->s_main, b);
  }
  CUDA_OK(cudaEventRecord(t1, c->s_main));
  double host_x = 0;
  CUDA_OK(cudaMemcpyAsync(&host_x, c->d_result, sizeof(double), cudaMemcpyDeviceToHost, c->s_main));
  if (dump_out && dump_table >= 0 && T[dump_table]) {
    const int W = (int)binom(k, pl.tables[dump_table].size);
    std::vector<char> raw((size_t)n * c->ld_of(W) * elem);
    CUDA_OK(cudaMemcpyAsync(raw.data(), T[dump_table], raw.size(), cudaMemcpyDeviceToHost, c->s_main));
    CUDA_OK(cudaStreamSynchronize(c->s_main));
    dump_out->assign((size_t)n * W, 0.0);
    for (int64_t v = 0; v < n; ++v)
      for (int j = 0; j < W; ++j) {
        const size_t off = (size_t)v * c->ld_of(W) + j;
        (*dump_out)[(size_t)v * W + j] =
            elem == 8 ? reinterpret_cast<double *>(raw.data())[off] : reinterpret_cast<float *>(raw.data())[off];
      }
  }
  if (root_out) {
    root_out->resize((size_t)n);
    if (n) CUDA_OK(cudaMemcpyAsync(root_out->data(), per_vertex, (size_t)n * 8, cudaMemcpyDeviceToHost, c->s_main));
  }
  for (int id = 0; id < nt; ++id) {
    c->afree(T[id], Tbytes[id], c->s_main);
    c->afree(Nb[id], Nbytes[id], c->s_main);
  }
  c->afree(hist, hist_bytes, c->s_main);
  if (per_vertex) {
    void *pv = per_vertex;
    c->afree(pv, (size_t)std::max<int64_t>(n, 1) * 8, c->s_main);
  }
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  if (c->opt.world > 1) CUDA_OK(cudaStreamSynchronize(c->s_comm));
  std::fill(c->prof, c->prof + PH_N + 1, 0.0);
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, t0, t1));
  c->prof[0] = ms;
  for (auto &e : c->ev_log) {
    float m = 0;
    CUDA_OK(cudaEventElapsedTime(&m, e.second.first, e.second.second));
    c->prof[1 + e.first] += m;
  }
  c->stats[4] = (double)c->peak_bytes;
  if (!std::isfinite(host_x)) throw Error(CC_ERR_NONFINITE, "colourful count is not finite (fp32 table overflow?)");
  *X = host_x;
}

cc_status fail(cc_ctx *c, const Error &e) {
  if (c) {
    c->err = e.what();
    if (e.status == CC_ERR_CUDA || e.status == CC_ERR_NCCL) c->poisoned = true;
  }
  return e.status;
}

#define API_BEGIN(c)                                                              \
  if (!(c)) return CC_ERR_ARG;                                                    \
  if ((c)->poisoned) {                                                            \
    (c)->err = "context poisoned by an earlier CUDA/NCCL error";                  \
    return CC_ERR_STATE;                                                          \
  }                                                                               \
  try {                                                                           \
    CUDA_OK(cudaSetDevice((c)->opt.device));
#define API_END(c)                                                                \
  }                                                                               \
  catch (const Error &e) {                                                        \
    return fail((c), e);                                                          \
  }                                                                               \
  catch (const std::bad_alloc &) {                                                \
    (c)->err = "host allocation failed";                                          \
    return CC_ERR_OOM;                                                            \
  }                                                                               \
  catch (const std::exception &e) {                                               \
    (c)->err = e.what();                                                          \
    return CC_ERR_ARG;                                                            \
  }                                                                               \
  (c)->err.clear();                                                               \
  return CC_OK;

}  // namespace

// ============================================================== C ABI
extern "C" {

cc_status cc_default_options(cc_options *opt) {
  if (!opt) return CC_ERR_ARG;
  std::memset(opt, 0, sizeof(*opt));
  opt->precision = CC_FP64;
  opt->world = 1;
  opt->use_graphs = 1;
  opt->relabel_seed = 0x5eed;
  return CC_OK;
}

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

cc_status cc_create(const cc_options *opt, cc_ctx **out) {
  if (!opt || !out) return CC_ERR_ARG;
  if (opt->precision != CC_FP64 && opt->precision != CC_FP32) return CC_ERR_ARG;
  if (opt->world < 1 || opt->world > 64 || opt->rank < 0 || opt->rank >= opt->world) return CC_ERR_ARG;
  if (opt->world > 1 && !opt->nccl_id) return CC_ERR_ARG;
  if (opt->chunk_cols < 0 || opt->segment_len < 0) return CC_ERR_ARG;
  std::unique_ptr<cc_ctx> c(new cc_ctx());
  c->opt = *opt;
  c->opt.nccl_id = nullptr;
  try {
    CUDA_OK(cudaSetDevice(opt->device));
    CUDA_OK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, opt->device));
    CUDA_OK(cudaStreamCreateWithFlags(&c->s_main, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, opt->device));
    uint64_t thr = UINT64_MAX;
    CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    c->n_partials = cc::dev::agg_partials_blocks(c->num_sms);
    c->d_partials = c->pmalloc<double>((size_t)c->n_partials);
    c->d_result = c->pmalloc<double>(1);
    if (opt->world > 1) {
      auto &api = cc::nccl();
      if (!api.ok) throw Error(CC_ERR_NCCL, api.why);
      ncclUniqueId id;
      std::memcpy(&id, opt->nccl_id, sizeof(id));
      NCCL_OK(api.CommInitRank(&c->comm, opt->world, id, opt->rank));
    }
  } catch (const Error &e) {
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
  if (c->comm) cc::nccl().CommDestroy(c->comm);
  for (void *p : c->persistent) cudaFree(p);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto e : c->ev_color)
    if (e) cudaEventDestroy(e);
  if (c->s_main) cudaStreamDestroy(c->s_main);
  if (c->s_comm) cudaStreamDestroy(c->s_comm);
  delete c;
}

const char *cc_last_error(const cc_ctx *c) { return c ? c->err.c_str() : "null context"; }

cc_status cc_load_graph(cc_ctx *c, int64_t n, const int64_t *row_ptr, const int32_t *col) {
  API_BEGIN(c)
  cc::HostGraph g = cc::validate_graph(n, row_ptr, col);
  // keep the scratch buffers, drop graph-dependent device state
  void *pr = c->d_partials, *rs = c->d_result;
  c->persistent.erase(std::remove_if(c->persistent.begin(), c->persistent.end(),
                                     [&](void *p) { return p == pr || p == rs; }),
                      c->persistent.end());
  bool had_template = c->has_template;
  free_graph(c);
  c->persistent.push_back(pr);
  c->persistent.push_back(rs);
  c->d_partials = static_cast<double *>(pr);
  c->d_result = static_cast<double *>(rs);
  c->part = cc::partition_graph(g, c->opt.world, c->opt.rank, c->opt.relabel_seed);
  const auto &R = c->part;
  c->n_global = n;
  c->n_own = R.n_own;
  c->n_halo = R.n_halo;
  c->n_rows = R.n_own + R.n_halo;
  c->d_rp = c->pupload(R.rp);
  c->d_col = c->pupload(R.col);
  std::vector<int32_t> orig(R.own_orig);
  orig.insert(orig.end(), R.halo_orig.begin(), R.halo_orig.end());
  orig.insert(orig.end(), R.iso_orig.begin(), R.iso_orig.end());
  c->n_crow = (int64_t)orig.size();
  c->d_orig = c->pupload(orig);
  c->d_colors = c->pmalloc<uint8_t>((size_t)std::max<int64_t>(c->n_crow, 1));
  std::vector<int64_t> beg(R.rp.begin(), R.rp.end() - (R.rp.empty() ? 0 : 1)), end(R.rp.begin() + (R.rp.empty() ? 0 : 1), R.rp.end());
  build_work(c, beg, end, false, c->w_full);  // world 1: the one pass; any world: the colour histogram
  if (c->opt.world > 1) {
    c->d_mid = c->pupload(R.mid);
    c->d_send_idx = c->pupload(R.send_idx);
    build_work(c, beg, R.mid, false, c->w_local);
    build_work(c, R.mid, end, true, c->w_remote);
  }
  c->has_graph = true;
  if (had_template) {
    upload_template(c);
    c->has_template = true;
  }
  c->has_colors = false;
  API_END(c)
}

cc_status cc_set_template(cc_ctx *c, int32_t k, const int32_t *parent) {
  API_BEGIN(c)
  c->plan = cc::make_plan(k, parent);
  upload_template(c);
  c->has_template = true;
  c->has_colors = false;
  API_END(c)
}

cc_status cc_color(cc_ctx *c, uint64_t seed) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_color needs a graph and a template");
  if (!c->ev_color[0]) {
    CUDA_OK(cudaEventCreate(&c->ev_color[0]));
    CUDA_OK(cudaEventCreate(&c->ev_color[1]));
  }
  CUDA_OK(cudaEventRecord(c->ev_color[0], c->s_main));
  cc::dev::launch_color(c->d_orig, c->n_crow, seed, c->plan.k, c->d_colors, c->s_main);
  c->check_launch();
  CUDA_OK(cudaEventRecord(c->ev_color[1], c->s_main));
  CUDA_OK(cudaStreamSynchronize(c->s_main));
  float ms = 0;
  CUDA_OK(cudaEventElapsedTime(&ms, c->ev_color[0], c->ev_color[1]));
  c->color_ms = ms;
  c->has_colors = true;
  API_END(c)
}

cc_status cc_set_colors(cc_ctx *c, const uint8_t *colors) {
  API_BEGIN(c)
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_set_colors needs a graph and a template");
  if (!colors && c->n_global) throw Error(CC_ERR_ARG, "colors is NULL");
  const auto &R = c->part;
  std::vector<uint8_t> h((size_t)c->n_crow);
  for (int64_t i = 0; i < R.n_own; ++i) h[i] = colors[R.own_orig[i]];
  for (int64_t i = 0; i < R.n_halo; ++i) h[R.n_own + i] = colors[R.halo_orig[i]];
  for (size_t i = 0; i < R.iso_orig.size(); ++i) h[c->n_rows + i] = colors[R.iso_orig[i]];
  for (auto x : h)
    if (x >= c->plan.k) throw Error(CC_ERR_ARG, "colour out of [0, k)");
  if (!h.empty()) CUDA_OK(cudaMemcpy(c->d_colors, h.data(), h.size(), cudaMemcpyHostToDevice));
  c->has_colors = true;
  API_END(c)
}

cc_status cc_get_colors(cc_ctx *c, uint8_t *colors) {
  API_BEGIN(c)
  if (!c->has_colors) throw Error(CC_ERR_STATE, "no colouring");
  if (c->opt.world != 1) throw Error(CC_ERR_STATE, "cc_get_colors needs world == 1");
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
  run_count(c, X, -1, nullptr, nullptr);
  API_END(c)
}

cc_status cc_estimate(cc_ctx *c, int32_t iterations, uint64_t seed0, double *estimate, double *per_iter) {
  API_BEGIN(c)
  if (iterations < 1 || !estimate) throw Error(CC_ERR_ARG, "iterations >= 1 and estimate != NULL required");
  if (!c->has_graph || !c->has_template) throw Error(CC_ERR_STATE, "cc_estimate needs a graph and a template");
  long double mean = 0;
  std::vector<double> xs((size_t)iterations);
  for (int j = 0; j < iterations; ++j) {
    cc::dev::launch_color(c->d_orig, c->n_crow, seed0 + (uint64_t)j, c->plan.k, c->d_colors, c->s_main);
    c->check_launch();
    c->has_colors = true;
    run_count(c, &xs[j], -1, nullptr, nullptr);
    mean += xs[j];
  }
  mean /= iterations;
  long double scale = 1;  // k^k / k!
  for (int i = 1; i <= c->plan.k; ++i) scale *= (long double)c->plan.k / i;
  *estimate = (double)(mean * scale / (long double)c->plan.aut);
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
  if (c->opt.world != 1) throw Error(CC_ERR_STATE, "cc_get_subtree_counts needs world == 1");
  const auto &pl = c->plan;
  if (x < 0 || x >= pl.k || !out) throw Error(CC_ERR_ARG, "bad template vertex or NULL output");
  const auto &R = c->part;
  const int tid = pl.full_table[x];
  double X = 0;
  if (tid == -2) {  // root: per-vertex C(v, T, [k])
    std::memset(out, 0, (size_t)c->n_global * sizeof(double));
    if (pl.k == 1) {
      for (int64_t v = 0; v < c->n_global; ++v) out[v] = 1.0;
    } else {
      std::vector<double> root;
      run_count(c, &X, -1, nullptr, &root);
      for (int64_t i = 0; i < R.n_own; ++i) out[R.own_orig[i]] = root[i];
    }
  } else if (tid == -1) {  // a leaf: the single-vertex table [S == {col v}]
    std::vector<uint8_t> h((size_t)c->n_crow);
    if (!h.empty()) CUDA_OK(cudaMemcpy(h.data(), c->d_colors, h.size(), cudaMemcpyDeviceToHost));
    std::memset(out, 0, (size_t)c->n_global * pl.k * sizeof(double));
    for (int64_t i = 0; i < R.n_own; ++i) out[(size_t)R.own_orig[i] * pl.k + h[i]] = 1.0;
    for (size_t i = 0; i < R.iso_orig.size(); ++i) out[(size_t)R.iso_orig[i] * pl.k + h[c->n_rows + i]] = 1.0;
  } else {
    std::vector<double> tab;
    run_count(c, &X, tid, &tab, nullptr);
    const int W = (int)cc::binom(pl.k, pl.tables[tid].size);
    std::memset(out, 0, (size_t)c->n_global * W * sizeof(double));
    for (int64_t i = 0; i < R.n_own; ++i)
      std::memcpy(out + (size_t)R.own_orig[i] * W, tab.data() + (size_t)i * W, (size_t)W * sizeof(double));
  }
  API_END(c)
}

cc_status cc_last_profile(cc_ctx *c, double *ms, int32_t cap, int32_t *n) {
  if (!c || !ms) return CC_ERR_ARG;
  const int m = std::min<int>(cap, PH_N + 1);
  for (int i = 0; i < m; ++i) ms[i] = c->prof[i];
  if (m > 1 + PH_COLOR) ms[1 + PH_COLOR] = c->color_ms;
  if (n) *n = m;
  return CC_OK;
}

cc_status cc_last_stats(cc_ctx *c, double *out, int32_t cap) {
  if (!c || !out || cap < 5) return CC_ERR_ARG;
  for (int i = 0; i < 5; ++i) out[i] = c->stats[i];
  return CC_OK;
}

// ---------------------------------------------------------------- host-only
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

}  // extern "C"
