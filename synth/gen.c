/*
 * synth/gen.c -- seeded synthetic INPUT generators (graphs only).
 *
 * This module is shared by the oracle side and the CUDA side as the single
 * source of test/bench inputs.  It holds none of the colour-coding method's
 * arithmetic: no colouring, no colour sets, no counting.  It only builds
 * simple undirected graphs in CSR form.
 *
 * Workloads stand in for the paper's datasets (Table 2, lines
 * 552-571: Twitter, Orkut, R-MAT "RMAT-250M/500M" with skew 1/3/8), which are
 * not available; BASELINE.json `configs` fixes the substitutes:
 *   - Erdos-Renyi G(n, m): m distinct edges drawn uniformly (config 0);
 *   - R-MAT (a, b, c, d) quadrant recursion, symmetrised, deduplicated and
 *     self-loops removed (configs 1-4).
 * DESIGN.md "Input recipe" states the readings (counter-based generator, one
 * 24-bit uniform per recursion level, no noise, no vertex relabel).
 *
 * Randomness: a counter-based generator (the "wyrand"-style 64-bit mixer
 * below, keyed by (seed, stream, counter)), so that the output depends only on
 * the arguments and not on thread scheduling.  CSR rows come out sorted.
 *
 * Memory: the caller receives a handle; `synth_graph_copy` copies the CSR
 * into caller buffers; `synth_graph_free` releases it.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
  int64_t n;
  int64_t nnz;      /* adjacency entries = 2 * undirected edges */
  int64_t *row_ptr; /* n + 1 */
  int32_t *col;     /* nnz, each row sorted ascending */
} synth_graph;

/* 64-bit mixer for the input generator (Moremur-style constants).  Distinct
 * from the colouring hash of the method on purpose. */
static inline uint64_t gmix(uint64_t x) {
  x ^= x >> 27;
  x *= 0x3C79AC492BA7B653ULL;
  x ^= x >> 33;
  x *= 0x1C69B3F74AC4AE35ULL;
  x ^= x >> 27;
  return x;
}
static inline uint64_t grand(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return gmix(gmix(seed * 0xD1342543DE82EF95ULL + stream) ^ (ctr + 0x632BE59BD9B4E019ULL));
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* Build a simple symmetric CSR from a directed edge list given by a callback
 * draw(i) -> (u, v), i in [0, m_draws).  Self-loops dropped, both directions
 * inserted, duplicates removed.  Deterministic regardless of threads. */
typedef void (*draw_fn)(const void *ctx, int64_t i, int32_t *u, int32_t *v);

static synth_graph *build_symmetric(int64_t n, int64_t m_draws, draw_fn draw, const void *ctx) {
  synth_graph *g = (synth_graph *)calloc(1, sizeof(synth_graph));
  if (!g) return NULL;
  g->n = n;
  int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt) { free(g); return NULL; }
  /* 1. degree count (with duplicates) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m_draws; ++i) {
    int32_t u, v;
    draw(ctx, i, &u, &v);
    if (u == v) continue;
    __atomic_fetch_add(&cnt[u], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&cnt[v], 1, __ATOMIC_RELAXED);
  }
  /* 2. prefix sum */
  int64_t *off = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
  off[0] = 0;
  for (int64_t v = 0; v < n; ++v) off[v + 1] = off[v] + cnt[v];
  int64_t total = off[n];
  int32_t *tmp = (int32_t *)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
  int64_t *cur = cnt; /* reuse as cursor */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) cur[v] = off[v];
  /* 3. fill (order nondeterministic; fixed by the per-row sort below) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m_draws; ++i) {
    int32_t u, v;
    draw(ctx, i, &u, &v);
    if (u == v) continue;
    int64_t pu = __atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED);
    int64_t pv = __atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED);
    tmp[pu] = v;
    tmp[pv] = u;
  }
  /* 4. sort + unique each row; new degree into cnt */
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; ++v) {
    int64_t b = off[v], e = off[v + 1];
    if (e - b > 1) qsort(tmp + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
    int64_t w = b;
    for (int64_t j = b; j < e; ++j)
      if (j == b || tmp[j] != tmp[j - 1]) tmp[w++] = tmp[j];
    cnt[v] = w - b;
  }
  /* 5. compact */
  g->row_ptr = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
  g->row_ptr[0] = 0;
  for (int64_t v = 0; v < n; ++v) g->row_ptr[v + 1] = g->row_ptr[v] + cnt[v];
  g->nnz = g->row_ptr[n];
  g->col = (int32_t *)malloc((size_t)(g->nnz > 0 ? g->nnz : 1) * sizeof(int32_t));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; ++v)
    memcpy(g->col + g->row_ptr[v], tmp + off[v], (size_t)cnt[v] * sizeof(int32_t));
  free(tmp);
  free(off);
  free(cnt);
  return g;
}

/* ---------------- R-MAT ---------------- */
typedef struct {
  int scale;
  uint32_t ta, tab, tabc; /* thresholds on a 24-bit uniform */
  uint64_t seed;
} rmat_ctx;

static void rmat_draw(const void *vctx, int64_t i, int32_t *pu, int32_t *pv) {
  const rmat_ctx *c = (const rmat_ctx *)vctx;
  uint32_t u = 0, v = 0;
  for (int l = 0; l < c->scale; ++l) {
    uint32_t r = (uint32_t)(grand(c->seed, (uint64_t)l, (uint64_t)i) >> 40); /* 24-bit uniform */
    uint32_t bu, bv;
    if (r < c->ta) { bu = 0; bv = 0; }
    else if (r < c->tab) { bu = 0; bv = 1; }
    else if (r < c->tabc) { bu = 1; bv = 0; }
    else { bu = 1; bv = 1; }
    u = (u << 1) | bu;
    v = (v << 1) | bv;
  }
  *pu = (int32_t)u;
  *pv = (int32_t)v;
}

/* R-MAT with 2^scale vertices and edge_factor * 2^scale directed draws. */
synth_graph *synth_rmat(int32_t scale, int32_t edge_factor, double a, double b, double c, uint64_t seed) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return NULL;
  rmat_ctx ctx;
  ctx.scale = scale;
  ctx.seed = seed;
  const double one = (double)(1u << 24);
  ctx.ta = (uint32_t)(a * one);
  ctx.tab = (uint32_t)((a + b) * one);
  ctx.tabc = (uint32_t)((a + b + c) * one);
  int64_t n = (int64_t)1 << scale;
  int64_t m = (int64_t)edge_factor << scale;
  return build_symmetric(n, m, rmat_draw, &ctx);
}

/* ---------------- Erdos-Renyi G(n, m) ---------------- */
typedef struct {
  const int32_t *eu, *ev;
} list_ctx;
static void list_draw(const void *vctx, int64_t i, int32_t *pu, int32_t *pv) {
  const list_ctx *c = (const list_ctx *)vctx;
  *pu = c->eu[i];
  *pv = c->ev[i];
}

/* m distinct undirected edges drawn uniformly over unordered pairs (rejection
 * of self-loops and repeats), in draw order.  Sequential (small n). */
synth_graph *synth_er(int64_t n, int64_t m, uint64_t seed) {
  if (n < 1 || n > (1LL << 31) - 1 || m < 0 || m > n * (n - 1) / 2) return NULL;
  int32_t *eu = (int32_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  int32_t *ev = (int32_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  /* open-addressing set of canonical pairs */
  int64_t cap = 16;
  while (cap < 4 * m + 16) cap <<= 1;
  uint64_t *set = (uint64_t *)malloc((size_t)cap * sizeof(uint64_t));
  for (int64_t i = 0; i < cap; ++i) set[i] = ~0ULL;
  int64_t got = 0;
  for (uint64_t ctr = 0; got < m; ++ctr) {
    uint64_t r = grand(seed, 7, ctr);
    uint64_t u = (uint64_t)(((unsigned __int128)(r & 0xFFFFFFFFULL) * (uint64_t)n) >> 32);
    uint64_t v = (uint64_t)(((unsigned __int128)(r >> 32) * (uint64_t)n) >> 32);
    if (u == v) continue;
    if (u > v) { uint64_t t = u; u = v; v = t; }
    uint64_t key = u * (uint64_t)n + v;
    uint64_t h = gmix(key) & (uint64_t)(cap - 1);
    int dup = 0;
    while (set[h] != ~0ULL) {
      if (set[h] == key) { dup = 1; break; }
      h = (h + 1) & (uint64_t)(cap - 1);
    }
    if (dup) continue;
    set[h] = key;
    eu[got] = (int32_t)u;
    ev[got] = (int32_t)v;
    ++got;
  }
  free(set);
  list_ctx lc = {eu, ev};
  synth_graph *g = build_symmetric(n, m, list_draw, &lc);
  free(eu);
  free(ev);
  return g;
}

/* Simple symmetric CSR from an explicit undirected edge list (both
 * directions are inserted; self-loops and duplicates removed). */
synth_graph *synth_from_edges(int64_t n, int64_t m, const int32_t *eu, const int32_t *ev) {
  list_ctx lc = {eu, ev};
  return build_symmetric(n, m, list_draw, &lc);
}

void synth_graph_size(const synth_graph *g, int64_t *n, int64_t *nnz) {
  *n = g->n;
  *nnz = g->nnz;
}
void synth_graph_copy(const synth_graph *g, int64_t *row_ptr, int32_t *col) {
  memcpy(row_ptr, g->row_ptr, ((size_t)g->n + 1) * sizeof(int64_t));
  if (g->nnz) memcpy(col, g->col, (size_t)g->nnz * sizeof(int32_t));
}
void synth_graph_free(synth_graph *g) {
  if (!g) return;
  free(g->row_ptr);
  free(g->col);
  free(g);
}

/* Uniform random colours as a plain input array (for cc_set_colors-style
 * tests where the colouring is passed in): out[v] = floor(u * k). */
void synth_uniform_u8(int64_t n, int32_t k, uint64_t seed, uint8_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v)
    out[v] = (uint8_t)(((grand(seed, 11, (uint64_t)v) >> 32) * (uint64_t)k) >> 32);
}
