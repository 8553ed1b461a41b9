// kernels.cuh -- device kernels of the colour-coding DP (sm_100a) and their
// host launchers.  Tables use the COLOUR-COMPRESSED row layout (DESIGN.md
// "Data layout"): the row of vertex v (colour c) of a sub-template of size t
// holds only the colour sets S that contain c -- the only ones that can be
// non-zero -- indexed by the colex rank of S' = sq_c(S \ {c}) in the
// (k-1)-colour universe (sq_c shifts colours above c down by one), i.e.
// C(k-1, t-1) entries.  Neighbour sums N''(v, Y'') are indexed by
// Y'' = sq_c(Y), |Y| = p, Y not containing c: C(k-1, p) entries.
// Storage type T = double (CC_FP64) or float (CC_FP32); neighbour sums and
// root products accumulate in double.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cc {
namespace dev {

// Implementation switches of the launchers (A/B knobs, not results: every
// setting computes the same values).  Read ONCE from the environment at
// cc_create (CC_<NAME>) and changeable per context with
// cc_set_knob; the defaults are the measured choices.
struct Knobs {
  int fused_root = 1;      // CC_FUSED_ROOT: 0 = never evaluate the root in an epilogue
  int sector_skip = 1;     // CC_SECTOR_SKIP: 0 = read every sector of a neighbour's row
  int gather_impl = 0;     // CC_GATHER_IMPL: 0 = by row width, 1 = rings only, 2 = lean only
  int narrow_impl = 4;     // CC_NARROW_IMPL: 4 = long lists row-parallel + short tail on rings, 0 = rings only,
                           //                 1 = row-parallel only
  int narrow_split = -1;   // CC_NARROW_SPLIT: log2(T/8), items with > T neighbours row-parallel; -1 = auto
  int csort_small = 1;     // CC_CSORT_SMALL: 0 = no separate kernel for the <= 8-neighbour items
  int combine_impl = 0;    // CC_COMBINE_IMPL: 0 = auto, 1 = Z-block, 2 = lane, 3 = V-tile, 4 = warp per vertex
  int acc32 = 1;           // CC_ACC32: fp32 tables keep the shared-memory N'' rows in fp32 (scaled)
  int phase_events = 1;    // CC_PHASE_EVENTS: per-kernel events for cc_last_profile
  int hub_l2_pct = 50;     // CC_HUB_L2_PCT: % of the L2 given an evict-last policy for hub rows (rings)
  int grid_reserve = -1;   // CC_GRID_RESERVE: SMs left free for NCCL while an exchange is in flight
                           //                  (-1 = auto: 8 when world > 1 over NCCL, else 0)
  int nvtx_mark = 0;       // CC_NVTX_MARK: i > 0 = the i-th neighbour-sum pass of a count runs inside
                           //               the NVTX range "cc_dominant" (one-launch ncu measurement)
  int short_lists = 2;     // CC_SHORT_LISTS: the short tail of wide-row gathers: 0 = with the long lists,
                           //   1 = k_gather_short, 2 = lean kernel U = 2 at 3 CTAs/SM (measured best),
                           //   3 = U = 1 at 4 CTAs/SM, 4 = U = 3 at 3 CTAs/SM
  int rows_variant = 0;    // CC_ROWS_VARIANT: row-parallel narrow kernel: 0 = U 4 at 3 CTAs/SM,
                           //   1 = U 2 at 4 CTAs/SM, 2 = U 8 at 2 CTAs/SM
  int short_split = 4;     // CC_SHORT_SPLIT: q, the short tail = light items with <= 8 << q neighbours
  int lean_split = -1;     // CC_LEAN_SPLIT: q >= 0 = wide-row gathers run as two launches, the items with
                           //   more than 8 << q neighbours and the rest (measurement of the short tail)
  int layout = 0;          // CC_LAYOUT: column order of tables of >= 3 vertices (R-3): 0 = colex;
                           //   L = 1, 2, 3: groups of 32 << (L-1) bytes whose sets share the most colours
  int tail_batches = 0;    // CC_TAIL_BATCHES: > 0 forces the memory plan's row batches (0 = by memory)
  int pair_gather = 0;     // CC_PAIR_GATHER: 1 = sibling narrow passives ready at the same time are summed
                           //   in one traversal (one rank); measured slower on configs[3] (33.7 ms for the
                           //   p = 2 + p = 3 pair against 25.1 ms unpaired, profiles/r2/SUMMARY.md)
  int combine_static = 1;  // CC_COMBINE_STATIC: the Z-block combines of (K; K-3, a') shapes with the
                           //   cover, columns and register indices fixed at compile time (combine_s.cu):
                           //   1 = K = 9 (configs[2]), 2 = also K = 11 (configs[3]; measured slower:
                           //   instruction-fetch bound), 0 = never
  int combine_zglobal = 1; // CC_COMBINE_ZGLOBAL: Z-block covers too large for shared memory (configs[4]'s
                           //   (7;4,3), 627 blocks) read from global memory (0: lane kernel instead)
  int combine_wreg = 1;    // CC_COMBINE_WREG: warp-per-vertex combines with 2-3 splits per output keep the
                           //   split pairs in registers (0: read them from shared memory per vertex)
  int wide_warps = 0;      // CC_WIDE_WARPS: > 0 = warps per CTA of the lean gather for N'' rows of > 8 KB
  int wide_nv = 4;         // CC_WIDE_NV: 16-byte vectors per lane per pass for rows of > 128 vectors (4 or 6)
  int tail_warps = 4;      // CC_TAIL_WARPS: warps per CTA of the lean gather's short-tail launch (72 registers:
                           //   7 CTAs of 4 warps = 28 warps per SM instead of 3 x 8 = 24)
  int tail_recompute_cols = 0;  // CC_TAIL_RECOMPUTE_COLS: > 0 forces the tail's passive to be recomputed
                                //   per batch in column chunks of this width (0 = by memory)
};

// Work list of one aggregation pass (Alg. 4: the
// neighbour list of a vertex is cut into tasks of at most s neighbours).
//   light[i]       vertices whose [beg, end) range has <= s neighbours
//   seg_*          segments of heavy vertices, grouped per heavy vertex
//   hv_first/nseg  first segment and segment count of heavy vertex h
// Items are numbered segments first, then light vertices.
struct AggWork {
  const int32_t *light = nullptr;
  int64_t n_light = 0;
  const int32_t *seg_v = nullptr;
  const int64_t *seg_b = nullptr, *seg_e = nullptr;
  const int32_t *seg_hv = nullptr;
  const int32_t *hv_first = nullptr, *hv_nseg = nullptr;
  int64_t n_seg = 0, n_hv = 0;
};

// Per-colouring descriptor of one work item (written by the colour sort):
// the item's neighbour stream is its colour-sorted range minus the group of
// the row vertex's own colour (those neighbours contribute nothing).
struct ItemDesc {
  int64_t b;      // first neighbour position of the item
  int32_t v;      // row vertex
  int32_t n_s;    // stream length = (e - b) - skip
  int32_t cv_lo;  // start of the own-colour group (relative to b)
  int32_t skip;   // size of the own-colour group
  int32_t cv;     // colour of v
  int32_t heavy;  // 1 for a heavy-vertex segment
};
static_assert(sizeof(ItemDesc) == 32, "ItemDesc is loaded as two 16-byte vectors");

struct GatherArgs {
  const int64_t *beg;     // per vertex: first neighbour position of this pass
  const int64_t *end;     // per vertex: one past the last
  const int32_t *col;     // neighbour ids, colour-sorted within each item
  const uint16_t *goff;   // per item: 16 cumulative colour-group end offsets (relative to item begin)
  const ItemDesc *desc;   // per item descriptor (bulk gather)
  const uint8_t *colors;  // colour of every row (owned | halo)
  const void *src;        // passive table P' (rows x ld_src): columns [col_base, col_base + W_in) of
  int64_t ld_src;         // the compressed rows (C(k-1, p-1) in all), src pointing at column col_base
  int W_in;
  int col_base = 0;       // column chunk: absolute index of src's first column, a multiple of 8
  int64_t item_from = 0;  // this launch takes items [item_from, item_to) (a row batch, or the
  int64_t item_to = -1;   // narrow kernels' split of the list); -1: all items
  int64_t item_split = 0; // first light item with <= 32 neighbours (items are in degree order)
  int64_t lean_split = -1; // knob lean_split: the lean kernel runs as two launches split at this item
  int64_t short_from = -1; // first light item with <= 32 neighbours (wide rows: the short-list kernel); -1: none
  const uint16_t *map;    // [c_u][c_v][map_ld] -> rank of Y'' in C(k-1, p), 0xFFFF = unusable
  int64_t map_ld;         // map row stride (multiple of 8 entries, padding = 0xFFFF)
  const uint32_t *skip = nullptr;  // [k-1][skip_words]: bit v of word w set = 16-byte vector 32 w + v of a
  int skip_words = 0;               // row lies in a 32-byte sector of sets that all contain that colour
  int64_t hub_rows;       // rows [0, hub_rows) of src are gathered with an L2 evict-last policy
  void *dst;              // N'' (rows x ld_dst), W_out = C(k-1, p)
  int64_t ld_dst;
  int W_out;
  int k;
  int accumulate;         // 0: dst = sum; 1: dst += sum
  double *scratch;        // n_seg x ld_scratch doubles (heavy partial rows)
  int64_t ld_scratch;
  unsigned int *arrive;   // n_hv counters (zeroed before launch)
  AggWork work;
  // Fused root (the root step's neighbour sum is needed nowhere else): the
  // epilogue does not write N'' but X_v = sum_{X'} A'(v, X') N''(v, comp X')
  // (Eq. 2 at the root + Eq. 3's summand) into per_vertex[v].
  int root_mode = 0;      // 0: write N''; 1: A' = table rA; 2: A' = N'' itself (root active = lift of this passive)
  const void *rA = nullptr;
  int64_t ldA = 0;
  int WA = 0;
  const uint16_t *comp = nullptr;  // comp[X'] = rank of [k-1] \ X' in C(k-1, p)
  double *per_vertex = nullptr;
  // Sibling pair (one rank, narrow rows; src2 != nullptr): a second passive
  // table summed in the SAME traversal of the colour-sorted lists (the two
  // neighbour sums of Eq. 1 over the same N(v)).  The
  // launch sees a virtual row of nvec1 16-byte vectors of part 1 (src, map,
  // skip) followed by part 2's (src2, map2, skip2); W_in = nvec1 x the vector
  // width + W_in2.  The virtual N'' row is part 1's o2 entries (written to
  // dst) followed by part 2's W_out - o2 entries (written to dst2).  No
  // column chunks, no fused root.
  const void *src2 = nullptr;
  int64_t ld_src2 = 0;
  int W_in2 = 0;
  int nvec1 = 0;
  const uint16_t *map2 = nullptr;
  int64_t map_ld2 = 0;
  const uint32_t *skip2 = nullptr;
  int skip_words2 = 0;
  void *dst2 = nullptr;
  int64_t ld_dst2 = 0;
  int o2 = 1 << 30;  // first N'' entry of part 2 (virtual row); unpaired: never reached
};

int launch_color(const int32_t *orig, int64_t n, uint64_t seed, int k, uint8_t *out, cudaStream_t s);
// out[i] = by_orig[orig[i]] for i < n; *bad |= 1 if a colour is >= k.
int launch_permute_colors(const uint8_t *by_orig, const int32_t *orig, int64_t n, int k, uint8_t *out, unsigned *bad,
                          cudaStream_t s);
// Colour-sort every item's neighbour range (stable) into col_out and record
// the 16 cumulative colour-group offsets of the item.
int launch_csort(const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                 const AggWork &work, int32_t *col_out, uint16_t *goff, ItemDesc *desc, int num_sms,
                 cudaStream_t s);
// World 1: the colour sort fused with the leaf level -- also writes
// N''(v, {y}) into hist (rows x ldh, k-1 columns) unless hist is null.
int launch_csort_hist(int elem, const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                      const AggWork &work, int k, int32_t *col_out, uint16_t *goff, ItemDesc *desc, void *hist,
                      int64_t ldh, int64_t hist_rows, int64_t small_from, const Knobs &kn, int num_sms,
                      cudaStream_t s);
// N''(v, {y}) = #{u in N(v) : sq_{c_v}(col u) = y}, k-1 columns.
int launch_hist(int elem, const int64_t *beg, const int64_t *end, const int32_t *col, const uint8_t *colors,
                const AggWork &work, int64_t n, int k, void *out, int64_t ld, int num_sms, cudaStream_t s);
// The neighbour sum of a passive table of size p >= 2 (compressed).
int launch_gather(int elem, const GatherArgs &a, const Knobs &kn, int num_sms, cudaStream_t s);
// Combine step; ztab (nullable) = its Z-block cover (zblock_table, nblocks
// blocks of zld entries) for the register-blocked kernel when combine_z_supported.
int launch_combine(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                   const uint32_t *split, int nq, int64_t n, void *out, int64_t ldO, int WO, const uint16_t *ztab,
                   int nblocks, int zld, int ts, int as, const Knobs &kn, int num_sms, cudaStream_t s);
bool combine_z_supported(int elem, int ts, int as);
// The compile-time-cover combine (combine_s.cu) for outputs of ts = K - 3
// colours of the compressed K-universe, fp32, colex columns; per_vertex !=
// nullptr = fused root (T' not stored, X_v written).  0 = shape unsupported.
int launch_combine_static(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN, int ts,
                          int as, int64_t n, void *out, int64_t ldO, double *per_vertex, const Knobs &kn, int num_sms,
                          cudaStream_t s);
// The combine restricted to the output columns [o_lo, o_hi) (a column chunk
// of the output table): out is the chunk's virtual base (column o
// of row v at out[v * ldO + o]); lane or V-tile kernel.
int launch_combine_cols(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                        const uint32_t *split, int nq, int64_t n, void *out, int64_t ldO, int WO, int o_lo, int o_hi,
                        const Knobs &kn, int num_sms, cudaStream_t s);
// The last combine fused with the root step that shares its passive table:
// X_v = sum_{X'} T'(v, X') N''(v, comp X') into per_vertex[v] (fp64), T'
// never stored.  Returns 0 (nothing launched) when the shape has no
// register-blocked kernel or its tile does not fit; the caller then runs the
// combine and launch_root.
int launch_combine_root(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN, int WN,
                        const uint16_t *ztab, int nblocks, int zld, int ts, int as, const uint16_t *comp, int64_t n,
                        double *per_vertex, const Knobs &kn, int num_sms, cudaStream_t s);
// Root step + deterministic reduction into result[0] (double).  A == nullptr
// means a single-vertex active part: sum_v N''(v, [k-1]) (one column).
int launch_root(int elem, const void *A, int64_t ldA, int WA, const void *N, int64_t ldN,
                const uint16_t *comp, int64_t n, double *partials, int n_partials, double *per_vertex,
                double *result, cudaStream_t s);
// X = sum_v sum_x R(v, x) for x < W (root of a template with fewer vertices
// than colours), per-vertex sums into per_vertex (nullable), result[0].
int launch_rowsum(int elem, const void *R, int64_t ld, int W, int64_t n, double *partials, int n_partials,
                  double *per_vertex, double *result, cudaStream_t s);
// Halo pack: out[i, 0:w) = src[idx[i], c0:c0+w) for i < rows (row strides ld / ldo;
// c0 and both strides multiples of the 16-byte vector; a ragged w is rounded
// up to whole vectors, reading the source row's padding).
int launch_pack(int elem, const void *src, int64_t ld, int64_t c0, int64_t w, const int32_t *idx, int64_t rows,
                void *out, int64_t ldo, cudaStream_t s);

int root_partials_blocks(int num_sms);  // grid size used by launch_root partials

}  // namespace dev
}  // namespace cc
