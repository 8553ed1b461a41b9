"""-m gpu: configs[4] (R-MAT scale 24, edge factor 64, 15-vertex perfect binary
tree, k = 15, fp32) at FULL size on ONE GPU.

The oracle cannot hold configs[4]'s tables (0.3-0.65 TB), so the
full-size run is pinned on sampled outputs the oracle computes one by one: the
B7 table row D_1(v, .) of the subtree at template vertex 1 (a depth-2 binary
tree) depends only on the 2-ball of v, so the oracle's fold-children DP on the
subgraph induced by that ball gives the exact row (BASELINE.json north_star:
"on sampled outputs the oracle can compute one by one").  The count itself is
checked for finiteness and for the fused root (self dot, mode 2) having run;
the whole-template parity of this path is the scaled twins' (test_gpu_parity).
"""
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_util import context, lib

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-4

# k = 16: the root with a leaf and two 7-vertex perfect binary subtrees -- a
# template whose 7-vertex subtree table alone (11.73 M rows x C(15, 6) fp64)
# is 470 GB and whose neighbour sum is 604 GB: it runs on ONE GPU only
# through the memory plan (row-batched tail, the subtree table recomputed per
# batch in column chunks).  fp64: at configs[4]'s hubs the neighbour sum of
# the 7-vertex subtree reaches ~1e42, beyond fp32 (reading C-13).  With the
# root's children in index order (fixed_root) the leaf is folded first, so
# the root step pairs the 9-vertex partial table with that neighbour sum.
PAR16 = [-1, 0, 0, 0, 2, 2, 4, 4, 5, 5, 3, 3, 10, 10, 11, 11]


@pytest.fixture(scope="module")
def graph4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return synth.CONFIGS[4].graph()


def ball(g, v, r):
    """Sorted vertex ids within distance r of v."""
    verts = np.array([v], dtype=np.int64)
    frontier = verts
    for _ in range(r):
        nxt = np.unique(np.concatenate([g.neighbors(int(u)) for u in frontier]))
        frontier = np.setdiff1d(nxt, verts)
        verts = np.union1d(verts, frontier)
    return verts


def induced(g, verts):
    """The subgraph induced by the sorted vertex ids `verts` (relabelled 0..)."""
    idx = -np.ones(g.n, dtype=np.int64)
    idx[verts] = np.arange(verts.size)
    eu, ev = [], []
    for i, x in enumerate(verts):
        nb = g.neighbors(int(x))
        j = idx[nb]
        keep = (j >= 0) & (j > i)
        eu.append(np.full(int(keep.sum()), i, dtype=np.int32))
        ev.append(j[keep].astype(np.int32))
    eu = np.concatenate(eu) if eu else np.zeros(0, np.int32)
    ev = np.concatenate(ev) if ev else np.zeros(0, np.int32)
    return synth.from_edges(int(verts.size), np.stack([eu, ev], axis=1))


def _sample_small_balls(g, want, max_ball, seed):
    deg = g.degrees()
    rng = np.random.default_rng(seed)
    cand = np.flatnonzero((deg >= 2) & (deg <= 6))
    rng.shuffle(cand)
    out = []
    for v in cand[:20000]:
        nb = g.neighbors(int(v))
        if 1 + nb.size + int(deg[nb].sum()) > max_ball:
            continue
        out.append(int(v))
        if len(out) == want:
            break
    return out


def test_config4_full_size_one_gpu_sampled_rows(graph4):
    cc = lib()
    cfg = synth.CONFIGS[4]
    g = graph4
    k = cfg.k
    seed = cfg.color_seed
    samples = _sample_small_balls(g, 6, 4000, 7)
    assert len(samples) >= 3, "no low-degree vertices with small 2-balls found"
    with context(g, cfg.parent, "fp32") as ctx:
        cc.cc_color(ctx, seed)
        x = cc.cc_count_colorful(ctx)
        st = cc.cc_last_stats(ctx)
        rows = cc.cc_get_subtree_rows(ctx, 1, samples, k, 7)
    assert math.isfinite(x) and x > 0
    assert st["fused_root"] == 2
    col = oracle.color(g.n, k, seed)
    for i, v in enumerate(samples):
        verts = ball(g, v, 2)
        sub = induced(g, verts)
        pos = int(np.searchsorted(verts, v))
        ref = oracle.dp_count(sub, cfg.parent, col[verts], oracle.NUM_DOUBLE, keep_x=1).table[pos]
        assert ref.shape == rows[i].shape
        zero = ref == 0
        assert np.all(rows[i][zero] == 0), f"v={v}: nonzero where the oracle has 0"
        if (~zero).any():
            err = np.max(np.abs(rows[i][~zero] - ref[~zero]) / ref[~zero])
            assert err <= TOL_FP32, f"v={v}: max rel err {err:.3e}"


def test_config4_template_on_the_clique_every_table_entry():
    """SURVEY 8(c) pin "Clique K_n, every table entry" with configs[4]'s own
    template (15-vertex perfect binary tree, k = 15) on K_2000 (4 M adjacency
    entries): D_x(v, S) = [c_v in S] (s - 1)! prod_{j in S, j != c_v} cnt_j
    for every template vertex x (subtree size s in {1, 3, 7}) and every S,
    and the root X_v = [k]'s entry; fp64 within 1e-12 per entry, fp32 X
    within 1e-4.  The fused root (self dot, mode 2) is on."""
    import itertools
    cc = lib()
    cfg = synth.CONFIGS[4]
    k, n = cfg.k, 2000
    g = synth.clique(n)
    col = oracle.color(n, k, 13)
    cnt = np.bincount(col, minlength=k).astype(np.float64)

    def closed(S, v):
        if col[v] not in S:
            return 0.0
        return math.factorial(len(S) - 1) * math.prod(cnt[j] - (j == col[v]) for j in S if j != col[v])

    verts = [0, 1, 777, 1999]
    with context(g, cfg.parent) as ctx:
        cc.cc_set_colors(ctx, col)
        x = cc.cc_count_colorful(ctx)
        assert cc.cc_last_stats(ctx)["fused_root"] == 2
        assert abs(x - math.factorial(k) * float(np.prod(cnt))) <= 1e-12 * x
        for xv, s in ((1, 7), (3, 3), (7, 1), (0, 15)):
            rows = cc.cc_get_subtree_rows(ctx, xv, verts, k, s)
            subsets = sorted(itertools.combinations(range(k), s), key=lambda t: t[::-1])
            for i, v in enumerate(verts):
                want = np.array([closed(S, v) for S in subsets])
                got = rows[i]
                assert np.all(got[want == 0] == 0), (xv, v)
                nz = want != 0
                assert np.max(np.abs(got[nz] - want[nz]) / want[nz]) <= 1e-12, (xv, v)
    with context(g, cfg.parent, "fp32") as ctx:
        cc.cc_set_colors(ctx, col)
        x32 = cc.cc_count_colorful(ctx)
    assert abs(x32 - math.factorial(k) * float(np.prod(cnt))) <= TOL_FP32 * x32


def test_star_closed_form_full_config4_graph(graph4):
    """SURVEY 8(c) star pin at full configs[4] scale (2.0 B adjacency
    entries, hubs of ~1 M neighbours): X(star with k-1 leaves) =
    (k-1)! sum_v prod_{j != c_v} cnt_j(v), k = 8, fp64 within 1e-12."""
    g = graph4
    k = 8
    col = oracle.color(g.n, k, 21)
    deg = g.degrees()
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    cnt = np.bincount(src * k + col[g.col], minlength=g.n * k).reshape(g.n, k).astype(np.float64)
    del src
    cnt[np.arange(g.n), col] = 1.0
    want = math.factorial(k - 1) * float(np.sum(np.prod(cnt, axis=1) * (deg > 0)))
    from gpu_util import count
    got = count(g, [-1] + [0] * (k - 1), seed=21, precision="fp64")
    assert abs(got - want) <= 1e-12 * want, (got, want)


def _root_samples(g, n, seed=7, max_ball2=20000, max_work=20_000_000):
    """n vertices (seeded order) of degree 4..12 whose radius-2 ball has at
    most max_ball2 vertices and degree sum at most max_work: the oracle's
    or_dp_root_at then costs seconds, however large the graph."""
    deg = g.degrees()
    cand = np.flatnonzero((deg >= 4) & (deg <= 12))
    np.random.default_rng(seed).shuffle(cand)
    out = []
    for v in cand[:200000]:
        nb = g.neighbors(int(v))
        if 1 + nb.size + int(deg[nb].sum()) > max_ball2:
            continue
        b2 = np.unique(np.concatenate([nb] + [g.neighbors(int(u)) for u in nb]))
        if int(deg[b2].sum()) > max_work:
            continue
        out.append(int(v))
        if len(out) == n:
            break
    return out


def _check_root_rows(got, want, what):
    for i, (x, w) in enumerate(zip(got, want)):
        if w == 0:
            assert x == 0, f"{what}: X_v = {x} where the oracle has 0 (sample {i})"
        else:
            assert abs(x - w) <= TOL_FP32 * abs(w), f"{what}: X_v = {x} vs oracle {w} (sample {i})"


def test_config4_full_size_root_counts(graph4):
    """configs[4] at full size, one GPU: the per-vertex root counts X_v (the
    summands of Eq. 3) of sampled vertices against the
    oracle's DP evaluated at that vertex (or_dp_root_at: the depth-3 template
    reads only the ball of radius 3), fp32 tables within 1e-4.  The fused
    root (self dot, mode 2) produced them."""
    cc = lib()
    cfg = synth.CONFIGS[4]
    g = graph4
    samples = _root_samples(g, 4)
    with context(g, cfg.parent, "fp32") as ctx:
        cc.cc_color(ctx, cfg.color_seed)
        rows = cc.cc_get_subtree_rows(ctx, 0, samples, cfg.k, cfg.k)[:, 0]
        assert cc.cc_last_stats(ctx)["fused_root"] == 2
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    want = [oracle.dp_root_at(g, cfg.parent, col, v, oracle.NUM_DOUBLE) for v in samples]
    assert any(w > 0 for w in want)
    _check_root_rows(rows, want, "configs[4] X_v")


def test_k16_template_with_7_vertex_subtrees_runs_on_one_gpu(graph4):
    """A k = 16 template (PAR16) on the configs[4] graph needs a 470 GB table
    of the 7-vertex subtree and a 604 GB neighbour sum (fp64) -- more than
    one GPU.  The memory plan runs it
    on ONE GPU: the tail of the plan in row batches, the 7-vertex subtree's
    table recomputed per batch in column chunks by its combine.  The count is
    finite and positive, the plan is the batched one within the device's
    memory, and sampled X_v equal the oracle's DP at those vertices (fp64,
    1e-12)."""
    cc = lib()
    g = graph4
    k = 16
    samples = _root_samples(g, 3)
    with context(g, PAR16, "fp64", fixed_root=1) as ctx:
        cc.cc_color(ctx, 2)
        rows = cc.cc_get_subtree_rows(ctx, 0, samples, k, k)[:, 0]  # one whole count, X_v kept
        st = cc.cc_last_stats(ctx)
        assert st["tail_batches"] >= 2 and st["recompute_cols"] > 0, st
        assert st["peak_table_bytes"] < 180e9
    assert np.all(np.isfinite(rows)) and np.all(rows >= 0)
    col = oracle.color(g.n, k, 2)
    want = [oracle.dp_root_at(g, PAR16, col, v, oracle.NUM_LONGDOUBLE) for v in samples]
    assert any(w > 0 for w in want)
    for i, (got, w) in enumerate(zip(rows, want)):
        assert abs(got - w) <= 1e-12 * abs(w) if w else got == 0, (i, got, w)
