/*
 * cc.h -- C ABI of the B200-native colour-coding hot path
 *         (Chen et al., "High-Performance Massive Subgraph Counting using
 *          Pipelined Adaptive-Group Communication", arXiv 1804.09764;
 *          cited as PAPER.md line numbers).
 *
 * Library: paper_1804_09764_b200/libcc.so (CUDA for sm_100a + C++ host code).
 * No torch types cross this boundary: plain host pointers and sizes.
 *
 * Problem: given a graph G and a tree
 * template T on k vertices, estimate #emb(T, G).  One colouring of G with k
 * colours is followed by the per-colouring dynamic
 * program of Eq. 1 / Eq. 2:
 *     C(v, T_i, S) = sum_{u in N(v)} sum_{S = S1 u S2} C(v, T_i', S1) * C(u, T_i'', S2)
 * computed here as "aggregate, then combine" (exact algebra):
 *     N(v, S2) = sum_{u in N(v)} C(u, T_i'', S2)          (SpMM-shaped gather)
 *     C(v, T_i, S) = sum_{(S1,S2) split of S} C(v, T_i', S1) * N(v, S2)
 * and the colourful total X = sum_v C(v, T, [k]) (Eq. 3 without its scale,
 * PAPER.md line 176).  Counting convention (reading C-1): the DP is
 * run with the over-count factor d = 1, so X counts colourful MAPS (injective
 * edge-preserving maps V_T -> V whose image is colourful); copies are
 * maps / |Aut(T)|.
 *
 * Conventions for every call:
 *  - Every call returns a cc_status; on failure cc_last_error(ctx) gives a
 *    message.  No C++ exception crosses the ABI.  Outputs are written only on
 *    CC_OK.
 *  - All pointer arguments are HOST memory.  The library copies inputs before
 *    returning, so the caller keeps ownership and may free them on return.
 *  - Device memory is owned by the context and released by cc_destroy.
 *  - After CC_ERR_CUDA or CC_ERR_NCCL the context is poisoned: every later
 *    call except cc_destroy / cc_last_error returns CC_ERR_STATE.
 *  - A context is bound to one CUDA device and is not thread-safe.
 *  - Multi-GPU (world > 1): one context per rank (one process per GPU).
 *    cc_load_graph, cc_set_template, cc_color, cc_set_colors,
 *    cc_count_colorful and cc_estimate are COLLECTIVE: all ranks call them in
 *    the same order with the same arguments (the same global CSR) and all
 *    ranks receive the same result.
 */
#ifndef CC_H
#define CC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cc_ctx cc_ctx; /* opaque, one per rank */

typedef enum {
  CC_OK = 0,
  CC_ERR_ARG = 1,       /* bad argument (null pointer, out-of-range option) */
  CC_ERR_GRAPH = 2,     /* CSR rejected by validation (see cc_load_graph) */
  CC_ERR_TEMPLATE = 3,  /* parent array is not a tree on 1..16 vertices */
  CC_ERR_STATE = 4,     /* call order violated, or context poisoned */
  CC_ERR_OOM = 5,       /* device or host allocation failed */
  CC_ERR_CUDA = 6,      /* CUDA runtime error (context poisoned) */
  CC_ERR_NCCL = 7,      /* NCCL error (context poisoned) */
  CC_ERR_NONFINITE = 8  /* fp32 tables overflowed: the result is not finite */
} cc_status;

/* Table precision (reading C-6; the paper states none). */
enum {
  CC_FP64 = 0, /* fp64 tables and accumulation: exact for integers < 2^53 */
  CC_FP32 = 1  /* fp32 table storage.  Neighbour sums: fp32 over blocks of at
                  most 32 neighbour rows of one colour group, the blocks added
                  into the vertex's N'' row held in shared memory in fp32
                  scaled by 2^-64 (acc32 knob, default; the short-list rings
                  sum blocks of 8 rows the same way) or fp64 (acc32 = 0);
                  heavy-segment partial rows and their
                  sum in fp64; combine split sums fp32 FMA; root products and
                  the final reduction fp64.  Worst-case relative error of X
                  ~8e-5 (reading C-6), measured 1e-10..1e-9 */
};

/* Halo-exchange schedule of the 1D partition (cc_options.exchange; PAPER.md
 * Alg. 3 "Adaptive-Group", lines 275-341). */
enum {
  CC_EXCHANGE_AUTO = 0,    /* pick by the pipeline cost model (cc_exchange_model),
                              the maximum over ranks, the same on every rank */
  CC_EXCHANGE_GROUPED = 1, /* one grouped send/recv with every peer (the
                              all-to-all branch, Alg. 3 line 15), overlapped with
                              the local neighbour sum, then one remote pass */
  CC_EXCHANGE_RING = 2,    /* world - 1 steps: step r sends to rank + r and
                              receives from rank - r (Alg. 3 lines 2-6), the
                              remote neighbour sum over step r's rows runs while
                              step r + 1 transfers (the pipeline, lines 326-341) */
  CC_EXCHANGE_ALLTOALL = 3, /* one ncclAlltoAll of per-peer blocks padded to the
                               largest send count of any rank pair, then the
                               blocks' rows moved into place */
  CC_EXCHANGE_DEVICE = 4    /* device-initiated: the pack kernel stores each
                               boundary row straight into the peer's halo window
                               (NCCL >= 2.28 symmetric window, LSA pointers over
                               NVLink, LSA barriers before and after); halo rows
                               in double-buffered chunk windows (as chunk_cols > 0);
                               needs a NCCL communicator (not loopback) */
};

typedef struct {
  int32_t precision;     /* CC_FP64 or CC_FP32 */
  int32_t device;        /* CUDA device ordinal for this rank */
  int32_t world;         /* number of ranks of the 1D vertex partition (>= 1) */
  int32_t rank;          /* this rank, 0 <= rank < world */
  const void *nccl_id;   /* 128-byte ncclUniqueId when world > 1 (from rank 0's
                            cc_nccl_unique_id, broadcast by the caller); ignored
                            when world == 1 */
  int64_t chunk_cols;    /* column chunks ("intermediate data
                            partitioning", lines 391-396 / 420-428 PeakMem): 0 =
                            none; > 0 = every neighbour sum reads its passive
                            table in launches of chunk_cols columns (rounded up
                            to a multiple of 8), the later ones accumulating into
                            N''; with world > 1 the halo rows are then exchanged
                            per chunk into two chunk-wide buffers (chunk i + 1
                            transfers while chunk i is summed) and tables keep
                            only the owned rows.  Independently of this option
                            the memory plan of every count runs the tail of the
                            plan in row batches, recomputing the tail's passive
                            table per batch in column chunks, when the tables
                            would not fit the free device memory (one rank).
                            < 0: CC_ERR_ARG */
  int32_t segment_len;   /* neighbour-list task size s: neighbour lists longer
                            than this are split into segments of at most s
                            neighbours (Alg. 4); 0 = auto */
  int32_t use_graphs;    /* 1: cc_count_colorful / cc_estimate (one rank)
                            replay a CUDA graph of the count's device work,
                            captured on first use and after any change of
                            graph, template, knobs or profiling (a new
                            colouring is data: the same graph); per-phase
                            profile times are then not reported.  For the
                            launch-bound small graphs (configs[0-1]); 0 or 1 */
  uint64_t relabel_seed; /* seed of the internal vertex permutation used to
                            balance the partition ("randomly
                            partitioned"); never changes results */
  int32_t fixed_root;    /* 0 = the planner picks the DP root and child order
                            minimising modelled bytes (the
                            root "can be picked arbitrarily"); 1 = root at the
                            parent -1 vertex, children in index order */
  int32_t replicas;      /* world > 1 only.  0 = 1D vertex partition (Alg. 2);
                            1 = colouring replicas (the
                            outer loop over colourings is parallel): every rank
                            keeps the whole graph, cc_count_colorful counts
                            locally (no exchange), and cc_estimate /
                            cc_estimate_mom run iteration j on rank j mod world
                            and all-reduce the per-iteration counts */
  void *loopback;        /* test hook, NULL for NCCL: a group from
                            cc_loopback_create -- the ranks are threads of one
                            process, possibly on one GPU; halo rows move with
                            event-ordered device copies, reductions on the
                            host (no kernel waits for another rank) */
  int32_t exchange;      /* CC_EXCHANGE_*; world > 1, replicas = 0 only */
} cc_options;

/* Fill *opt with defaults: CC_FP64, device 0, world 1, rank 0, auto sizes,
 * relabel_seed 0x5eed, planner-chosen root, 1D partition (replicas 0). */
cc_status cc_default_options(cc_options *opt);

/* Test hook: an in-process group of `world` ranks for cc_options.loopback
 * (each rank a host thread with its own context); destroy after every
 * context of the group. */
cc_status cc_loopback_create(int32_t world, void **group);
void cc_loopback_destroy(void *group);

/* Rank 0 only: write a fresh 128-byte ncclUniqueId to out128 (host).
 * CC_ERR_NCCL if libnccl.so.2 cannot be loaded. */
cc_status cc_nccl_unique_id(void *out128);

/* Create a context on opt->device.  For world > 1 this joins the NCCL
 * communicator (collective over all ranks).  *out receives the handle. */
cc_status cc_create(const cc_options *opt, cc_ctx **out);

/* Release all device memory, streams and the communicator.  NULL is a no-op. */
void cc_destroy(cc_ctx *ctx);

/* Message of the last failure on ctx ("" if none).  Valid until the next call. */
const char *cc_last_error(const cc_ctx *ctx);

/* Load the graph G (neighbour lists N(v)).
 *  n       : number of vertices, 0 <= n < 2^31
 *  row_ptr : n+1 int64 offsets, row_ptr[0] == 0, nondecreasing
 *  col     : row_ptr[n] int32 neighbour ids in [0, n)
 * The CSR must describe a simple undirected graph: no self-loops, no
 * duplicate neighbours within a row, and symmetric (u in N(v) <=> v in N(u)).
 * Rows need not be sorted.  Violations are REJECTED with CC_ERR_GRAPH (the
 * library never cleans input).  Internally: isolated vertices are dropped
 * from the tables (their rows are zero for templates of >= 2 vertices),
 * vertices are relabelled (hubs first per rank; seeded shuffle across ranks)
 * and, for world > 1, cut into balanced contiguous ranges with halo lists.
 * Invalidates the colouring. */
cc_status cc_load_graph(cc_ctx *ctx, int64_t n, const int64_t *row_ptr, const int32_t *col);

/* Set the tree template T as a parent array of k
 * entries, 1 <= k <= 16, exactly one -1 (the root rho(T));
 * every other entry is the index of the vertex's parent and the pointers must
 * form one tree.  Builds the sub-template partition (PAPER.md lines 110-113,
 * 122, 159: cut an edge at the root; the active part keeps the root, the
 * passive part is rooted at the cut neighbour), merges isomorphic
 * sub-templates, and uploads the colour-set split tables.  k colours are used
 * (PAPER.md line 154).  Invalidates the colouring.  CC_ERR_TEMPLATE on a bad
 * parent array. */
cc_status cc_set_template(cc_ctx *ctx, int32_t k, const int32_t *parent);

/* cc_set_template with a colouring of `colours` >= k colours (the
 * paper fixes colours = k): tables are indexed by colour
 * sets of the colours-universe, X sums the root table over every colour set
 * of size k, and the estimators divide by P(colourful) = colours! /
 * ((colours - k)! colours^k).  cc_set_template(ctx, k, parent) is
 * cc_set_template_colors(ctx, k, parent, k).  CC_ERR_ARG unless
 * k <= colours <= 16. */
cc_status cc_set_template_colors(cc_ctx *ctx, int32_t k, const int32_t *parent, int32_t colours);

/* Colour every vertex uniformly at random with k colours (PAPER.md lines
 * 156-158), on the device, from the shared seed and the ORIGINAL vertex id:
 *   col(v) = ((mix(mix(seed) ^ v) >> 32) * k) >> 32,
 *   mix = SplitMix64 finaliser (reading C-2).
 * Requires a template (k).  */
cc_status cc_color(cc_ctx *ctx, uint64_t seed);

/* Run the per-colouring DP (Alg. 1 lines 8-10, Eq. 2) and return
 * X = sum_v C(v, T(rho), [k]) -- the number of colourful maps for the current
 * colouring (Eq. 3 WITHOUT the k^k/k! scale).  In CC_FP64 mode X is exact
 * while below 2^53.  Requires graph, template and colouring
 * (CC_ERR_STATE otherwise).  CC_ERR_NONFINITE if fp32 tables overflowed. */
cc_status cc_count_colorful(cc_ctx *ctx, double *colorful_maps);

/* The estimator (Alg. 1 lines 4-13 and Eq. 3; DESIGN.md readings
 * C-1, C-10): for j = 0..iterations-1, colour with seed0 + j, count X_j, and
 * return *estimate = mean_j(X_j) * k^k / k! / |Aut(T)|, an estimate of the
 * number of non-induced copies of T.  per_iter (nullable) receives the
 * `iterations` values X_j.  iterations >= 1. */
cc_status cc_estimate(cc_ctx *ctx, int32_t iterations, uint64_t seed0, double *estimate,
                      double *per_iter);

/* Several templates on the current colouring (graphlet frequencies,
 * PAPER.md lines 46-50): X[i] = colourful maps of template i
 * (sizes[i] vertices, its parent array at parents + sizes[0] + ... +
 * sizes[i-1]) for the colouring set by cc_color / cc_set_colors, whose
 * colours (cc_set_template_colors) must be >= every sizes[i].  Isomorphic
 * rooted sub-templates are computed once across the templates, and so are
 * the neighbour sums of such passive parts (both kept while they fit a
 * quarter of the free device memory), the colour sort and the leaf level;
 * out[9] of cc_last_stats then gives the number of tables and sums reused.  One GPU (or replica mode).  The context's own template is
 * restored afterwards. */
cc_status cc_count_colorful_multi(cc_ctx *ctx, int32_t n_templates, const int32_t *sizes, const int32_t *parents,
                                  double *X);

/* The paper's estimator (Alg. 1 last line, lines 180-181): run
 * `iterations` colourings with seeds seed0 + j, form C_j = X_j k^k/k!/|Aut(T)|,
 * split them in iteration order into `groups` groups of equal size (the
 * remainder one per group from the front), and return the median of the
 * group means (mean of the two middle ones for an even count).  groups = 1
 * is cc_estimate.  per_iter (nullable) receives the X_j.  Collective.
 * Errors: CC_ERR_ARG unless 1 <= groups <= iterations. */
cc_status cc_estimate_mom(cc_ctx *ctx, int32_t iterations, uint64_t seed0, int32_t groups, double *estimate,
                          double *per_iter);

/* ---- test and bench hooks (off the hot path) ---------------------------- */

/* Use a caller-supplied colouring: colors[v] in [0, k) for every ORIGINAL
 * vertex id v < n (host array of n bytes; copied to the device). */
cc_status cc_set_colors(cc_ctx *ctx, const uint8_t *colors);

/* Copy the current colouring back, indexed by original vertex id (n bytes). */
cc_status cc_get_colors(cc_ctx *ctx, uint8_t *colors);

/* |Aut(T)|, |Aut_rho(T)| (automorphisms fixing the root) and the number of
 * DP steps of the plan. */
cc_status cc_template_info(cc_ctx *ctx, int64_t *aut, int64_t *aut_root, int32_t *n_steps);

/* Re-run the DP for the current colouring keeping every table, and copy the
 * full-subtree table of template vertex x, D_x(v, S), to out: n rows (ORIGINAL
 * vertex order) x C(k, s_x) columns (colex order of S), as double, where s_x is
 * the size of x's subtree.  For x = root this is the per-vertex C(v, T, [k]).
 * World must be 1. */
cc_status cc_get_subtree_counts(cc_ctx *ctx, int32_t x, double *out);

/* Row-sampled variant of cc_get_subtree_counts (test hook for graphs whose
 * full tables do not fit host memory): out[i * C(k, s) + r] = C(vertices[i],
 * T_x, S_r) for the nv ORIGINAL vertex ids given, same colex layout; the root
 * (x = parent -1 vertex) gives one column.  Runs one colouring's DP with the
 * user's rooting; the fused root stays on (the sampled rows are copied right
 * after their table is produced).  world == 1 only.  Errors: CC_ERR_ARG (bad
 * x / id / pointer), CC_ERR_STATE. */
cc_status cc_get_subtree_rows(cc_ctx *ctx, int32_t x, const int32_t *vertices, int32_t nv, double *out);

/* Implementation knobs (A/B switches of the launchers; every setting
 * computes the same values): name is one of fused_root, sector_skip,
 * gather_impl, narrow_impl, narrow_split, csort_small, combine_impl, acc32,
 * phase_events, hub_l2_pct, grid_reserve, tail_batches, tail_recompute_cols,
 * layout, nvtx_mark (meanings and defaults: DESIGN.md
 * section 9a).  Each context reads CC_<NAME> from the environment ONCE, in
 * cc_create; these calls change or read the context's value.  CC_ERR_ARG on
 * an unknown name or a NULL pointer.  Not collective: set the same value on
 * every rank. */
cc_status cc_set_knob(cc_ctx *ctx, const char *name, int32_t value);
cc_status cc_get_knob(cc_ctx *ctx, const char *name, int32_t *value);

/* Per-kernel timing events on (1, default) or off (0): off, cc_last_profile
 * reports only the total and the colouring, and cc_last_stats the bytes but
 * not the longest gather launch; small graphs then run without the event
 * records between their kernels (configs[0]: 0.042 -> 0.026 ms). */
cc_status cc_set_profiling(cc_ctx *ctx, int32_t on);

/* Timing of the last cc_count_colorful, in ms, per phase (device events):
 * out[0] = total, then colour, colour sort, leaf level, gathers, combines,
 * root, exchange (comm stream), exposed exchange (main-stream wait for halo
 * rows).  *n receives the number written. */
cc_status cc_last_profile(cc_ctx *ctx, double *ms, int32_t cap, int32_t *n);

/* Stats of the last cc_count_colorful: out[0] = U = sum over aggregations of
 * adjacency entries x columns ("edge x colour-set updates"),
 * out[1] = algorithmic bytes moved (model bytes), out[2] = algorithmic bytes
 * of the aggregation kernels alone, out[3] = number of kernel launches,
 * out[4] = peak table bytes, out[5] (cap >= 6) = fused-root mode of the
 * last count (0: none, 1: root dot with the active table, 2: self dot with
 * the lifted neighbour sum -- both in the last gather's epilogue; 3: root dot
 * in the epilogue of the combine that produces the root's active table), out[6] / out[7] (cap >= 8) = algorithmic bytes
 * and device ms of the longest neighbour-sum pass, out[8] = number of
 * neighbour-sum passes (a narrow-row pass is one or two kernels), out[9] = halo bytes received by this rank (1D
 * partition), out[10] (cap >= 11) = the exchange schedule in use
 * (0: none -- one rank or replicas, CC_EXCHANGE_GROUPED, CC_EXCHANGE_RING),
 * out[11] (cap >= 12) = column-chunk launches of the chunked neighbour sums
 * (0: none), out[12] = row batches of the memory plan's tail (0: none),
 * out[13] = column width of the tail's recomputed passive table (0: none),
 * out[14] (cap >= 15) = 1-based ordinal of the longest neighbour-sum pass
 * among the count's passes (the knob nvtx_mark selects a pass by it),
 * out[15] (cap >= 16) = sibling pairs: narrow neighbour sums taken along in
 * the traversal of another (one rank; knob pair_gather).
 * cap >= 5. */
cc_status cc_last_stats(cc_ctx *ctx, double *out, int32_t cap);

/* Test hook: the device-initiated exchange's machinery on a one-rank NCCL
 * communicator: a symmetric window (ncclMemAlloc + ncclCommWindowRegister),
 * a device communicator with LSA barriers (ncclDevCommCreate), and a kernel
 * that stores through ncclGetLsaPointer, syncs the barrier and reads the
 * values back.  CC_ERR_NCCL when the device API is missing or a value is
 * wrong. */
cc_status cc_nccl_device_selftest(int32_t device);

/* Test hook: a one-rank NCCL communicator on `device` runs the calls the
 * partitioned path uses -- a grouped ncclSend/ncclRecv (to itself) and an
 * fp64 ncclAllReduce -- and checks the values moved.  CC_ERR_NCCL when NCCL
 * cannot be loaded or a value is wrong, CC_ERR_CUDA on a device error. */
cc_status cc_nccl_selftest(int32_t device);

/* ---- host-only introspection (no GPU needed; used by CPU tests) --------- */

/* Median of means of n colourful counts X (as cc_estimate_mom, no GPU). */
cc_status cc_median_of_means(const double *X, int32_t n, int32_t k, int64_t aut, int32_t groups, double *out);

/* Niter = ceil(constant * e^k * ln(1/delta) / eps^2), at least 1 (PAPER.md
 * Alg. 1 line 3, line 154: Niter = O(e^k log(1/delta) / eps^2); the constant
 * is the caller's).  CC_ERR_ARG unless eps > 0, 0 < delta <= 1, k >= 1,
 * constant > 0. */
cc_status cc_niter(double eps, double delta, int32_t k, double constant, int64_t *out);

/* Colex rank of the colour set `mask` (bit c = colour c) among sets of the
 * same size: rank(S) = sum_i C(s_i, i+1), s_0 < s_1 < ... (combinatorial
 * number system).  Returns -1 on a bad argument. */
int64_t cc_colex_rank(uint32_t mask);

/* Inverse: the size-s set of rank r (k-independent); 0xFFFFFFFF if invalid. */
uint32_t cc_colex_unrank(int32_t s, int64_t r);

/* Split table of a step (t; a, p) with k colours: for every S of size t
 * (colex rank r < C(k,t)) and every q < C(t,a), the q-th subset S1 of S of
 * size a (colex over positions in S) and S2 = S \ S1, packed as
 * rank(S1) | rank(S2) << 16, stored at out[q * C(k,t) + r].  cap = entries
 * available in out.  CC_ERR_ARG if too small. */
cc_status cc_split_table(int32_t k, int32_t t, int32_t a, uint32_t *out, int64_t cap);

/* The Z-block cover of a combine step (outputs of size ts, actives of size
 * as, passives of size ts - as, in a K-colour universe) used by the
 * register-blocked combine: *n_blocks blocks of *ld uint16 entries each --
 * the colex ranks of the block's C(ts+1, as) active sets and C(ts+1, ts-as)
 * passive sets (local colex order) and of its ts+1 outputs Z \ {z}
 * (0xFFFF = owned by another block).  out may be NULL to query the sizes;
 * CC_ERR_ARG if cap is too small. */
cc_status cc_zblock_table(int32_t K, int32_t ts, int32_t as, uint16_t *out, int64_t cap, int32_t *n_blocks,
                          int32_t *ld);

/* Plan a template without a context.  steps_out receives, per step, 6 int32:
 * t, a, p, active table id (-1 = single vertex), passive table id (-1 = single
 * vertex), output table id (-1 = root).  Also |Aut(T)|, |Aut_rho(T)|, and
 * Table-3 memory = sum C(k,t), computation = sum C(k,t) C(t,a) over the
 * non-root steps. */
cc_status cc_plan_template(int32_t k, const int32_t *parent, int32_t *steps_out, int32_t cap_steps,
                           int32_t *n_steps, int64_t *aut, int64_t *aut_root, double *memory,
                           double *computation);

/* The plan cc_set_template would choose with fixed_root = 0 for a graph of
 * average degree avg_degree and elem-byte table entries (4 or 8): same
 * outputs as cc_plan_template plus *root = the chosen DP root and *cost = its
 * modelled bytes per stored vertex. */
cc_status cc_plan_template_auto(int32_t k, const int32_t *parent, double avg_degree, int32_t elem,
                                int32_t *steps_out, int32_t cap_steps, int32_t *n_steps, int32_t *root,
                                double *cost);

/* Partition plan of the 1D vertex partition (Alg. 2 line 2 and lines
 * 374-382) for rank `rank` of `world`, computed on the host exactly as
 * cc_load_graph does.  sizes_out[0..3] = n_own, n_halo, local CSR entries,
 * total send rows.  When the array pointers are non-NULL they receive:
 *   own_orig[n_own]   original ids of owned vertices, in internal order
 *   halo_orig[n_halo] original ids of halo vertices, in internal order
 *   recv_off[world+1] halo rows received from each peer (offsets into halo)
 *   send_off[world+1] offsets into send_idx per peer
 *   send_idx[...]     owned local indices sent to each peer, in the peer's
 *                     receive order
 *   rp[n_own+1], col[...] the local CSR; col < n_own is an owned row,
 *                     col >= n_own is halo row col - n_own.
 * Call once with NULL arrays to get sizes. */
cc_status cc_partition_plan(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t world,
                            int32_t rank, uint64_t relabel_seed, int64_t *sizes_out,
                            int32_t *own_orig, int32_t *halo_orig, int64_t *recv_off,
                            int64_t *send_off, int32_t *send_idx, int64_t *rp, int32_t *lcol);

/* The exchange cost model behind CC_EXCHANGE_AUTO for rank `rank` of `world`
 * (host only; the partition as cc_partition_plan): out[0] = modelled seconds
 * of one neighbour sum of a table with `row_bytes`-byte rows under the
 * grouped schedule, out[1] = under the ring pipeline, out[2] / out[3] = the
 * link and gather rates assumed (bytes/s).  cc_load_graph takes the maximum
 * of each over the ranks and runs the ring when it is below the grouped
 * figure. */
cc_status cc_exchange_model(int64_t n, const int64_t *row_ptr, const int32_t *col, int32_t world, int32_t rank,
                            uint64_t relabel_seed, double row_bytes, double *out);

#ifdef __cplusplus
}
#endif

#endif /* CC_H */
