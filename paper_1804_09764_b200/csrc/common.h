// common.h -- internal host-side types of libcc (not part of the C ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cc.h"

namespace cc {

// Thrown inside the library, converted to a cc_status at the ABI boundary.
struct Error : std::runtime_error {
  cc_status status;
  Error(cc_status s, const std::string &m) : std::runtime_error(m), status(s) {}
};

constexpr int kMaxK = 16;

// ---------------------------------------------------------------- colex.cpp
// Binomial coefficients C(n, r) for n, r <= 16 (exact in int64).
int64_t binom(int n, int r);
// Combinatorial number system (colex) rank / unrank of colour sets.
int64_t colex_rank(uint32_t mask);
uint32_t colex_unrank(int s, int64_t r);
// Split table of (t; a, t-a) over k colours: out[q * C(k,t) + r] =
// rank(S1) | rank(S2) << 16 for the q-th size-a subset S1 of S = unrank(t, r).
std::vector<uint32_t> split_table(int k, int t, int a);
// Lift (drop) table for a = 1: out[r * 16 + c] = rank(S \ {c}) for S = unrank(t, r)
// if c in S, else 0xFFFF.
std::vector<uint16_t> drop_table(int k, int t);
// Complement table at the root: out[r] = rank([k] \ X) for X = unrank(a, r).
std::vector<uint16_t> complement_table(int k, int a);
// Colour-compressed layout: sq_c removes colour c
// from the universe (higher colours shift down), us_c re-inserts it.
uint32_t squeeze(uint32_t mask, int c);
uint32_t unsqueeze(uint32_t mask, int c);
// Storage order of a table's compressed columns (build decision R-3): rank[q]
// = colex rank of the colour set at storage position q, pos = its inverse.
struct Layout {
  std::vector<int32_t> rank, pos;
};
Layout pack_layout(int K, int s, int E);  // sector-homogeneous order (E sets per 32-byte sector)
Layout identity_layout(int K, int s);

// Gather map of a passive part of size p: for neighbour colour cu, vertex
// colour cv and compressed index r of u's row (Y' = unrank(p-1, r) in the
// (k-1)-universe of cu), out[(cu*k + cv) * C(k-1,p-1) + r] = rank of
// sq_cv({cu} u us_cu(Y')) in C(k-1, p), or 0xFFFF if that set contains cv.
// With layouts: lin = the passive table's (input positions), lout = the
// neighbour sum's (output positions); nullptr = colex order.
std::vector<uint16_t> gather_map(int k, int p, const Layout *lin = nullptr, const Layout *lout = nullptr);
// Sector-skip table of a passive part of size p (rows of C(k-1, p-1) entries
// of elem bytes): for each colour c' of the (k-1)-universe, bit (vi mod 32)
// of word (vi / 32) marks 16-byte vector vi of a row whose whole 32-byte
// sector holds only sets containing c' (or padding) -- entries no
// destination of that colour can use.  *words receives the words per colour.
std::vector<uint32_t> skip_table(int k, int p, int elem, int *words, const Layout *lin = nullptr);
int64_t gather_map_ld(int k, int p);  // map row stride: C(k-1,p-1) rounded up to 8 (padding 0xFFFF)

// Z-block cover of a combine step with outputs of size ts = t-1, actives of
// size as = a-1 and passives of size ps = ts - as, in a K = k-1 colour
// universe: every output set lies in some block Z of ts + 1 colours, and all
// splits of all outputs inside Z use only the C(ts+1, as) active sets and
// C(ts+1, ps) passive sets of Z (the combine keeps Z's passive values in
// registers).  Per block, zblock_ld(ts, as) uint16 entries: the global colex
// ranks of Z's active sets (local colex order), of its passive sets, and of
// the output Z minus its z-th colour for each z (0xFFFF when another block
// owns that output).  *n_blocks receives the block count.
std::vector<uint16_t> zblock_table(int K, int ts, int as, int *n_blocks);
int64_t zblock_ld(int ts, int as);

// ---------------------------------------------------------------- plan.cpp
// One DP step (t; a, p): T_out(v, S) = sum_{S1 u S2 = S} A(v, S1) N_P(v, S2),
// N_P(v, S2) = sum_{u in N(v)} P(u, S2).  Table ids index Plan::tables;
// id -1 = the single-vertex table C(v, {x}, {c}) = [c == col v] (implicit).
struct Step {
  int t, a, p;
  int active;   // table id or -1
  int passive;  // table id or -1
  int out;      // table id, or -1 for the root step (t == k)
};

struct TableInfo {
  int size;       // number of template vertices = colour-set size
  int template_x; // a template vertex whose full subtree (or partial) this is
  int j;          // number of children of template_x included
  std::string code;
};

struct Plan {
  int k = 0;           // template vertices
  int kc = 0;          // colours (>= k); 0 = k
  int colours() const { return kc ? kc : k; }
  int root = -1;       // root of the plan (chosen by the planner)
  int user_root = -1;  // the parent -1 vertex of the user's array
  std::vector<int> parent;
  std::vector<Step> steps;
  std::vector<TableInfo> tables;
  int64_t aut = 1, aut_root = 1;
  double memory = 0, computation = 0;  // Table 3 quantities
  // Per template vertex x: table id of its full subtree (-1 for leaves = single vertex;
  // -2 for the root, whose table is the root step).
  std::vector<int> full_table;
  // Liveness: last step index that reads table id as active / as passive source.
  std::vector<int> table_last_use;
  // For each table id used as passive with p >= 2: first step (aggregation point)
  // and last step that consumes its aggregated N.
  std::vector<int> n_first_use, n_last_use;
};

// Planner options.  auto_root: choose the root and child order minimising
// plan_cost (the count of colourful maps does not depend on them, reading
// C-4); otherwise the root is the parent -1 vertex, children in index order.
struct PlanOpts {
  bool auto_root = true;
  double avg_degree = 32.0;  // adjacency entries per stored vertex
  int elem = 4;              // table entry bytes
  double fma_bytes = 4.0;    // weight of one combine FMA in bytes (measured: the combine
                             // kernels run ~1.5-4 TFMA/s against ~7 TB/s of gather bytes)
  int kc = 0;                // colours (0 = template size)
};
Plan make_plan(int k, const int32_t *parent, const PlanOpts *opts = nullptr);  // throws Error(CC_ERR_TEMPLATE)
double plan_cost(const Plan &P, const PlanOpts &o);

// ---------------------------------------------------------------- graph.cpp
// Validated CSR (copy) of the global graph.
struct HostGraph {
  int64_t n = 0, nnz = 0;
  const int64_t *rp = nullptr;  // n + 1 offsets: the caller's array (read only), valid during the call
  const int32_t *col = nullptr; // nnz ids: the caller's array when every row is sorted, else col_own
  std::vector<int64_t> rp_own;  // (n == 0: {0})
  std::vector<int32_t> col_own; // a sorted copy, only when some row was not sorted
  HostGraph() = default;
  HostGraph(HostGraph &&) = default;
  HostGraph(const HostGraph &) = delete;
};
// Validate (throws Error(CC_ERR_GRAPH)); the caller's arrays are used in
// place (no copy of a multi-GB CSR per rank) unless a row must be sorted.
HostGraph validate_graph(int64_t n, const int64_t *row_ptr, const int32_t *col);

// The 1D vertex partition of one rank (Alg. 2 line 2; lines 374-382).
struct RankPart {
  int world = 1, rank = 0;
  int64_t n_own = 0, n_halo = 0;
  std::vector<int32_t> own_orig;   // internal owned index -> original id
  std::vector<int32_t> halo_orig;  // halo index -> original id
  std::vector<int64_t> rp;         // local CSR over owned rows (n_own + 1)
  std::vector<int32_t> col;        // < n_own: owned row; >= n_own: halo row
  std::vector<int64_t> mid;        // first halo neighbour position per owned row
  std::vector<int64_t> recv_off;   // world + 1, offsets into halo rows
  std::vector<int64_t> send_off;   // world + 1, offsets into send_idx
  std::vector<int32_t> send_idx;   // owned local indices, per peer in receive order
  int64_t n_global = 0;            // n of the input graph (incl. isolated)
  std::vector<int32_t> iso_orig;   // isolated vertices (coloured, never in tables)
};
RankPart partition_graph(const HostGraph &g, int world, int rank, uint64_t relabel_seed);

// Per-peer split of every owned row's halo range: the neighbours of row i
// owned by peer q (Alg. 3's per-step set N_{r,w}(v))
// are positions [b[q * n_own + i], b[(q + 1) * n_own + i]) of the local CSR;
// q = world is rp[i + 1].  (world + 1) x n_own entries.
std::vector<int64_t> peer_bounds(const RankPart &R);

// Modelled time of one neighbour sum of a table with `row_bytes`-byte rows
// on this rank under the two exchange schedules (Alg. 3 and the
// pipeline analysis, lines 326-341, 420-441): grouped = one all-to-all of
// the halo rows overlapped with the local part, then one remote pass;
// ring = P - 1 steps (send to rank + r, receive from rank - r), the remote
// pass of step r overlapping the transfer of step r + 1.
struct ExchangeModel {
  double grouped_s = 0, ring_s = 0;
  double link_bps = 0, gather_bps = 0;
};
ExchangeModel model_exchange(const RankPart &R, const std::vector<int64_t> &bounds, double row_bytes);

}  // namespace cc
