/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * colour-coding hot path of Chen et al., arXiv 1804.09764 ("PAPER.md").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product (paper_1804_09764_b200/) never links, imports or calls it, and it
 * shares no code with the CUDA path: its own colouring hash, its own subset
 * indexing (enumeration lookup tables, no combinatorial arithmetic), its own
 * graph traversal.
 *
 * What it computes (reading C-1):
 *   X(G, T, col) = #{ f : V_T -> V injective, (x,y) in E_T => (f x, f y) in E,
 *                     col o f injective }                       (colourful maps)
 * -- PAPER.md lines 86-92 (non-induced embedding), 105-108 (colourful),
 * line 154 (k = |V_T| colours).  Two independent algorithms:
 *   or_brute_count : the definition, enumerated by DFS (exact, u128).
 *   or_dp_count    : the paper's recurrence, Eq. 1,
 *                    with d = 1 and the passive part always a whole child
 *                    subtree ("fold children"): for template vertex x with
 *                    children y_1..y_j, start from C(v,{x},{col v}) = 1 and for
 *                    each child y:  C'(v, S u Y) += C(v, S) * sum_{u in N(v)} D_y(u, Y)
 *                    over disjoint S, Y ("S = S1 u S2").
 *                    X = sum_v D_root(v, [k])   (Eq. 3 without the k^k/k!
 *                    scale).
 *   or_dp_root_at  : or_dp_count's DP at one root vertex v0 (its tables
 *                    evaluated only within each template vertex's depth of
 *                    v0): the summand X_v0 of Eq. 3, for sampled outputs of
 *                    graphs too large for the whole DP (pinned: sum over v0
 *                    = brute force, and = or_dp_count's per-vertex root).
 *   or_color       : reading C-2 (SplitMix64 finaliser; PAPER.md lines
 *                    156-158 only say "uniformly at random").
 *   or_estimate    : mean_j X_j * k^k/k! / |Aut(T)| (PAPER.md lines 146-147,
 *                    176; reading C-1 divides maps by |Aut(T)|; reading C-10
 *                    takes the mean).
 *   or_mom         : median of means (Alg. 1 last line, lines
 *                    180-181): C_j = X_j k^k/k!/|Aut(T)|, t groups of equal
 *                    size in iteration order (remainder one per group from
 *                    the front), median of the group
 *                    means (mean of the middle two for even t).
 *   or_niter       : Niter = ceil(c e^k ln(1/delta) / eps^2), >= 1 (Alg. 1
 *                    line 3; constant c = 1 by default,
 *                    SPEC.md lines 441-446).
 *   or_aut         : |Aut(T)| = #injective edge-preserving maps T -> T
 *                    (brute force of the definition on G = T).
 * Numeric types of the DP: exact unsigned __int128 with overflow detection,
 * long double, or double (reading C-6).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

typedef unsigned __int128 u128;

enum { OR_OK = 0, OR_EARG = 1, OR_EOVERFLOW = 2, OR_ENOMEM = 3 };

/* ------------------------------------------------------------------ */
/* Colouring (reading C-2).                                            */
/* ------------------------------------------------------------------ */
uint64_t or_mix(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void or_color(int64_t n, int32_t k, uint64_t seed, uint8_t *out) {
  uint64_t s = or_mix(seed);
  for (int64_t v = 0; v < n; ++v) {
    uint64_t h = or_mix(s ^ (uint64_t)v) >> 32;
    out[v] = (uint8_t)((h * (uint64_t)k) >> 32);
  }
}

/* ------------------------------------------------------------------ */
/* Template (parent array) helpers.                                    */
/* ------------------------------------------------------------------ */
typedef struct {
  int k, root;
  int parent[16];
  int nchild[16];
  int child[16][16]; /* children in increasing index order */
  int size[16];      /* subtree size */
  int post[16];      /* post-order (children before parent) */
  int depth[16];     /* distance from the root */
  int bfs[16];       /* BFS order from the root */
} tmpl;

static int tmpl_init(tmpl *t, int k, const int32_t *parent) {
  if (k < 1 || k > 16) return OR_EARG;
  memset(t, 0, sizeof(*t));
  t->k = k;
  t->root = -1;
  for (int i = 0; i < k; ++i) {
    t->parent[i] = parent[i];
    if (parent[i] == -1) {
      if (t->root >= 0) return OR_EARG;
      t->root = i;
    } else if (parent[i] < 0 || parent[i] >= k || parent[i] == i) {
      return OR_EARG;
    }
  }
  if (t->root < 0) return OR_EARG;
  for (int i = 0; i < k; ++i)
    if (parent[i] >= 0) t->child[parent[i]][t->nchild[parent[i]]++] = i;
  /* BFS from root; must reach all k vertices (connected tree) */
  int head = 0, tail = 0;
  t->bfs[tail++] = t->root;
  while (head < tail) {
    int x = t->bfs[head++];
    for (int c = 0; c < t->nchild[x]; ++c) {
      if (tail >= k) return OR_EARG;
      t->bfs[tail++] = t->child[x][c];
    }
  }
  if (tail != k) return OR_EARG; /* a cycle in the parent pointers */
  for (int i = 1; i < k; ++i) t->depth[t->bfs[i]] = t->depth[t->parent[t->bfs[i]]] + 1;
  /* post-order = reverse BFS works as "children before parent" */
  for (int i = 0; i < k; ++i) t->post[i] = t->bfs[k - 1 - i];
  for (int i = 0; i < k; ++i) t->size[i] = 1;
  for (int i = 0; i < k; ++i) {
    int x = t->post[i];
    if (t->parent[x] >= 0) t->size[t->parent[x]] += t->size[x];
  }
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Brute force: enumerate maps of the definition.                      */
/* ------------------------------------------------------------------ */
typedef struct {
  const int64_t *rp;
  const int32_t *col;
  const uint8_t *colors; /* NULL -> count all injective maps */
  const tmpl *t;
  int32_t img[16];
} bf_state;

static u128 bf_dfs(bf_state *s, int depth) {
  const tmpl *t = s->t;
  if (depth == t->k) return 1;
  int x = t->bfs[depth];
  int32_t pv = s->img[t->parent[x]];
  u128 total = 0;
  for (int64_t e = s->rp[pv]; e < s->rp[pv + 1]; ++e) {
    int32_t u = s->col[e];
    int ok = 1;
    for (int d = 0; d < depth && ok; ++d) {
      int32_t w = s->img[t->bfs[d]];
      if (w == u) ok = 0;
      else if (s->colors && s->colors[w] == s->colors[u]) ok = 0;
    }
    if (!ok) continue;
    s->img[x] = u;
    total += bf_dfs(s, depth + 1);
  }
  return total;
}

/* mode: 1 = colourful maps (needs colors), 0 = all injective maps. */
int or_brute_count(int64_t n, const int64_t *rp, const int32_t *col, int32_t k,
                   const int32_t *parent, const uint8_t *colors, int32_t mode,
                   uint64_t *out_lo, uint64_t *out_hi) {
  tmpl t;
  int rc = tmpl_init(&t, k, parent);
  if (rc) return rc;
  if (mode == 1 && !colors) return OR_EARG;
  u128 total = 0;
#pragma omp parallel
  {
    u128 mine = 0;
    bf_state s;
    s.rp = rp;
    s.col = col;
    s.colors = mode == 1 ? colors : NULL;
    s.t = &t;
#pragma omp for schedule(dynamic, 16)
    for (int64_t v = 0; v < n; ++v) {
      s.img[t.root] = (int32_t)v;
      mine += bf_dfs(&s, 1);
    }
#pragma omp critical
    total += mine;
  }
  *out_lo = (uint64_t)total;
  *out_hi = (uint64_t)(total >> 64);
  return OR_OK;
}

/* |Aut(T)| = injective edge-preserving maps T -> T. */
int or_aut(int32_t k, const int32_t *parent, uint64_t *out) {
  tmpl t;
  int rc = tmpl_init(&t, k, parent);
  if (rc) return rc;
  /* the template as a symmetric CSR */
  int64_t rp[17];
  int32_t col[32];
  int deg[16] = {0};
  for (int i = 0; i < k; ++i)
    if (parent[i] >= 0) { deg[i]++; deg[parent[i]]++; }
  rp[0] = 0;
  for (int i = 0; i < k; ++i) rp[i + 1] = rp[i] + deg[i];
  int fill[16] = {0};
  for (int i = 0; i < k; ++i)
    if (parent[i] >= 0) {
      int p = parent[i];
      col[rp[i] + fill[i]++] = p;
      col[rp[p] + fill[p]++] = i;
    }
  uint64_t lo, hi;
  rc = or_brute_count(k, rp, col, k, parent, NULL, 0, &lo, &hi);
  if (rc) return rc;
  *out = lo;
  return hi ? OR_EOVERFLOW : OR_OK;
}

/* ------------------------------------------------------------------ */
/* Subset indexing by enumeration: masks of each size in increasing     */
/* integer order; rank_of[mask] = position in that list.               */
/* ------------------------------------------------------------------ */
typedef struct {
  int k;
  int32_t *rank_of;   /* 2^k */
  int32_t *masks[17]; /* masks[s][i], i < count[s] */
  int64_t count[17];
} subsets;

static int subsets_init(subsets *ss, int k) {
  memset(ss, 0, sizeof(*ss));
  ss->k = k;
  int64_t full = (int64_t)1 << k;
  ss->rank_of = (int32_t *)malloc((size_t)full * sizeof(int32_t));
  if (!ss->rank_of) return OR_ENOMEM;
  for (int s = 0; s <= k; ++s) ss->count[s] = 0;
  for (int64_t m = 0; m < full; ++m) ss->count[__builtin_popcountll((unsigned long long)m)]++;
  for (int s = 0; s <= k; ++s) {
    ss->masks[s] = (int32_t *)malloc((size_t)ss->count[s] * sizeof(int32_t));
    if (!ss->masks[s]) return OR_ENOMEM;
  }
  int64_t fill[17] = {0};
  for (int64_t m = 0; m < full; ++m) {
    int s = __builtin_popcountll((unsigned long long)m);
    ss->rank_of[m] = (int32_t)fill[s];
    ss->masks[s][fill[s]++] = (int32_t)m;
  }
  return OR_OK;
}
static void subsets_free(subsets *ss) {
  free(ss->rank_of);
  for (int s = 0; s <= ss->k; ++s) free(ss->masks[s]);
}

/* ------------------------------------------------------------------ */
/* The fold-children DP, instantiated for three numeric types.          */
/* ------------------------------------------------------------------ */
#define NUM u128
#define SFX u128
#define EXACT 1
#include "dp_body.inc"
#undef NUM
#undef SFX
#undef EXACT

#define NUM long double
#define SFX ld
#define EXACT 0
#include "dp_body.inc"
#undef NUM
#undef SFX
#undef EXACT

#define NUM double
#define SFX f64
#define EXACT 0
#include "dp_body.inc"
#undef NUM
#undef SFX
#undef EXACT

#define NUM u128
#define SFX u128
#define EXACT 1
#include "dp_root_body.inc"
#undef NUM
#undef SFX
#undef EXACT
#define NUM long double
#define SFX ld
#define EXACT 0
#include "dp_root_body.inc"
#undef NUM
#undef SFX
#undef EXACT
#define NUM double
#define SFX f64
#define EXACT 0
#include "dp_root_body.inc"
#undef NUM
#undef SFX
#undef EXACT

/* One row of the combine step of Eq. 1 in double:
 *   T(S u Y) += A(S) * N(Y)  for |S| = a, |Y| = p, S and Y disjoint,
 * rows indexed by colex rank (= increasing-mask order).  Exposed so the
 * worked example of Fig. 1b can be checked on the
 * same code the DP uses. */
int or_combine_row(int32_t k, int32_t a, int32_t p, const double *A, const double *N, double *T) {
  if (k < 1 || k > 16 || a < 1 || p < 1 || a + p > k) return OR_EARG;
  subsets ss;
  if (subsets_init(&ss, k)) { subsets_free(&ss); return OR_ENOMEM; }
  int of = 0;
  combine_row_f64(&ss, a, p, A, N, T, &of);
  subsets_free(&ss);
  return OR_OK;
}

/* kc >= k colours (PAPER.md line 146 fixes kc = k): tables are
 * indexed by colour sets of the kc-colour universe and the total sums the
 * root table over every colour set of size k.
 * numtype: 0 = exact u128 (OR_EOVERFLOW on overflow), 1 = long double, 2 = double.
 * keep_x: template vertex whose full-subtree table D_x(v, S) is written to
 *   out_table (n x C(k, size_x), colex order; as double), or -1.
 * out_root: if non-NULL, per-vertex D_root(v, [k]) as double (n entries).
 * Total X: exact in (out_lo, out_hi) for numtype 0; as long double in *out_ld. */
int or_dp_count_kc(int64_t n, const int64_t *rp, const int32_t *col, int32_t k,
                   const int32_t *parent, const uint8_t *colors, int32_t kc, int32_t numtype,
                   int32_t keep_x, double *out_table, double *out_root,
                   uint64_t *out_lo, uint64_t *out_hi, long double *out_ld) {
  tmpl t;
  int rc = tmpl_init(&t, k, parent);
  if (rc) return rc;
  if (keep_x >= k || keep_x < -1 || kc < k || kc > 16) return OR_EARG;
  for (int64_t v = 0; v < n; ++v)
    if (colors[v] >= kc) return OR_EARG;
  subsets ss;
  if (subsets_init(&ss, kc)) { subsets_free(&ss); return OR_ENOMEM; }
  switch (numtype) {
    case 0: {
      u128 tot = 0;
      rc = dp_u128(&ss, &t, n, rp, col, colors, keep_x, out_table, out_root, &tot);
      if (!rc) { *out_lo = (uint64_t)tot; *out_hi = (uint64_t)(tot >> 64); if (out_ld) *out_ld = (long double)tot; }
      break;
    }
    case 1: {
      long double tot = 0;
      rc = dp_ld(&ss, &t, n, rp, col, colors, keep_x, out_table, out_root, &tot);
      if (!rc && out_ld) *out_ld = tot;
      break;
    }
    case 2: {
      double tot = 0;
      rc = dp_f64(&ss, &t, n, rp, col, colors, keep_x, out_table, out_root, &tot);
      if (!rc && out_ld) *out_ld = (long double)tot;
      break;
    }
    default:
      rc = OR_EARG;
  }
  subsets_free(&ss);
  return rc;
}

/* The root's count at ONE vertex v0, D_root(v0, [k]) (the summand of Eq. 3
 * at v0), for graphs too large for the whole DP: the same fold-children
 * recurrence, where the table of a template vertex at depth d is kept only
 * for the vertices within distance d of v0 -- exactly the rows the root at
 * v0 reads (a child's row at u is read by its parent at a neighbour of u).
 * Vertices are numbered in BFS order from v0, so those rows are a prefix.
 * Exact total in (out_lo, out_hi) for numtype 0, else *out_ld. */
int or_dp_root_at(int64_t n, const int64_t *rp, const int32_t *col, int32_t k, const int32_t *parent,
                  const uint8_t *colors, int32_t numtype, int64_t v0, uint64_t *out_lo, uint64_t *out_hi,
                  long double *out_ld) {
  tmpl t;
  int rc = tmpl_init(&t, k, parent);
  if (rc) return rc;
  if (v0 < 0 || v0 >= n) return OR_EARG;
  int h = 0;
  for (int x = 0; x < k; ++x) h = t.depth[x] > h ? t.depth[x] : h;
  /* BFS from v0 to depth h: queue order; end[d] = number of vertices within distance d */
  int32_t *dist = (int32_t *)malloc((size_t)n * sizeof(int32_t));
  int32_t *qpos = (int32_t *)malloc((size_t)n * sizeof(int32_t));
  int64_t cap = 1024, len = 0;
  int32_t *queue = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
  if (!dist || !qpos || !queue) { free(dist); free(qpos); free(queue); return OR_ENOMEM; }
  for (int64_t v = 0; v < n; ++v) dist[v] = -1;
  int64_t end[17] = {0};
  dist[v0] = 0;
  queue[len++] = (int32_t)v0;
  for (int64_t head = 0; head < len; ++head) {
    const int32_t v = queue[head];
    if (dist[v] >= h) continue;
    for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
      const int32_t u = col[e];
      if (dist[u] >= 0) continue;
      dist[u] = dist[v] + 1;
      if (len == cap) {
        cap *= 2;
        int32_t *q2 = (int32_t *)realloc(queue, (size_t)cap * sizeof(int32_t));
        if (!q2) { free(dist); free(qpos); free(queue); return OR_ENOMEM; }
        queue = q2;
      }
      queue[len++] = u;
    }
  }
  for (int64_t i = 0; i < len; ++i) {
    qpos[queue[i]] = (int32_t)i;
    end[dist[queue[i]]] = i + 1;
  }
  for (int d = 1; d <= h; ++d) if (end[d] < end[d - 1]) end[d] = end[d - 1];
  subsets ss;
  if (subsets_init(&ss, k)) { subsets_free(&ss); free(dist); free(qpos); free(queue); return OR_ENOMEM; }
  switch (numtype) {
    case 0: {
      u128 x = 0;
      rc = droot_u128(&ss, &t, rp, col, colors, queue, qpos, end, &x);
      if (!rc) { *out_lo = (uint64_t)x; *out_hi = (uint64_t)(x >> 64); if (out_ld) *out_ld = (long double)x; }
      break;
    }
    case 1: {
      long double x = 0;
      rc = droot_ld(&ss, &t, rp, col, colors, queue, qpos, end, &x);
      if (!rc && out_ld) *out_ld = x;
      break;
    }
    case 2: {
      double x = 0;
      rc = droot_f64(&ss, &t, rp, col, colors, queue, qpos, end, &x);
      if (!rc && out_ld) *out_ld = (long double)x;
      break;
    }
    default:
      rc = OR_EARG;
  }
  subsets_free(&ss);
  free(dist);
  free(qpos);
  free(queue);
  return rc;
}

int or_dp_count(int64_t n, const int64_t *rp, const int32_t *col, int32_t k,
                const int32_t *parent, const uint8_t *colors, int32_t numtype,
                int32_t keep_x, double *out_table, double *out_root,
                uint64_t *out_lo, uint64_t *out_hi, long double *out_ld) {
  return or_dp_count_kc(n, rp, col, k, parent, colors, k, numtype, keep_x, out_table, out_root, out_lo, out_hi,
                        out_ld);
}

/* Median of means (Alg. 1 last line, lines 180-181). */
static int cmp_ld(const void *a, const void *b) {
  const long double x = *(const long double *)a, y = *(const long double *)b;
  return x < y ? -1 : x > y;
}
double or_mom(int32_t iters, const double *X, int32_t k, uint64_t aut, int32_t t) {
  if (iters < 1 || t < 1 || t > iters) return -1.0;
  long double scale = 1;
  for (int i = 1; i <= k; ++i) scale *= (long double)k / i; /* k^k / k! */
  long double *Z = (long double *)malloc(sizeof(long double) * (size_t)t);
  int pos = 0;
  for (int g = 0; g < t; ++g) {
    const int size = iters / t + (g < iters % t ? 1 : 0);
    long double s = 0;
    for (int j = 0; j < size; ++j) s += (long double)X[pos + j] * scale / (long double)aut;
    pos += size;
    Z[g] = s / size;
  }
  qsort(Z, (size_t)t, sizeof(long double), cmp_ld);
  const long double med = t % 2 ? Z[t / 2] : (Z[t / 2 - 1] + Z[t / 2]) / 2;
  free(Z);
  return (double)med;
}

/* Niter = ceil(c e^k ln(1/delta) / eps^2), at least 1 (Alg. 1 line 3). */
int64_t or_niter(double eps, double delta, int32_t k, double c) {
  if (!(eps > 0) || !(delta > 0) || !(delta <= 1) || k < 1 || !(c > 0)) return -1;
  const double v = ceil(c * exp((double)k) * log(1.0 / delta) / (eps * eps));
  return v < 1 ? 1 : (int64_t)v;
}

/* Estimator (Alg. 1, lines 146-147 and 176; readings C-1, C-10):
 * mean_j X_j * k^k / k! / aut. */
double or_estimate(int32_t iters, const double *X, int32_t k, uint64_t aut) {
  long double mean = 0;
  for (int j = 0; j < iters; ++j) mean += X[j];
  mean /= iters;
  long double scale = 1;
  for (int i = 1; i <= k; ++i) scale *= (long double)k / i; /* k^k / k! */
  return (double)(mean * scale / (long double)aut);
}
