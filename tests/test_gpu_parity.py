"""-m gpu: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * colouring: bit-exact (integer work);
  * fp64 mode: every table entry within relative 1e-12, zero entries exactly
    zero; bit-exact on configs[0] (integers < 2^53);
  * fp32 mode: final colourful count within relative 1e-4.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_close_entries, context, count, lib, rel_err, subtree_sizes, tables

pytestmark = pytest.mark.gpu

TOL_FP64 = 1e-12
TOL_FP32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def oracle_tables(g, parent, col, numtype):
    k = len(parent)
    out = {}
    sizes = subtree_sizes(parent)
    for x in range(k):
        if parent[x] == -1:
            r = oracle.dp_count(g, parent, col, numtype, want_root=True)
            out[x] = r.root.reshape(-1, 1)
        else:
            out[x] = oracle.dp_count(g, parent, col, numtype, keep_x=x).table
        assert out[x].shape[1] == math.comb(k, sizes[x] if parent[x] != -1 else k)
    return out


# ------------------------------------------------------------------ colouring
def test_colouring_bit_exact_vs_oracle():
    cc = lib()
    for n, k, seed in ((1000, 5, 2), (65_536, 7, 2), (1_000_003, 12, 123456789), (70_000, 16, 2 ** 63 + 5)):
        g = synth.cycle(n)
        with context(g, list(range(-1, k - 1))) as ctx:
            cc.cc_color(ctx, seed)
            got = cc.cc_get_colors(ctx, n)
        assert np.array_equal(got, oracle.color(n, k, seed)), (n, k, seed)


def test_colouring_includes_isolated_vertices():
    cc = lib()
    g = synth.from_edges(10, [(0, 1), (5, 6)])
    with context(g, [-1, 0, 1]) as ctx:
        cc.cc_color(ctx, 9)
        assert np.array_equal(cc.cc_get_colors(ctx, 10), oracle.color(10, 3, 9))


# ------------------------------------------------------------------ configs[0]: bit-exact
def test_config0_bit_exact_count_and_every_table():
    cfg = synth.CONFIGS[0]
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_EXACT).total
    assert count(g, cfg.parent, seed=cfg.color_seed) == float(want)
    got = tables(g, cfg.parent, col)
    ref = oracle_tables(g, cfg.parent, col, oracle.NUM_EXACT)
    for x in range(cfg.k):
        assert np.array_equal(got[x], ref[x]), f"table of template vertex {x}"


# ------------------------------------------------------------------ small-graph suite, exact
def _small_suite():
    rng = np.random.default_rng(1234)
    cases = []
    for trial in range(30):
        k = int(rng.integers(2, 9))
        n = int(rng.integers(k, 40))
        g = synth.gnp(n, float(rng.choice([0.1, 0.3, 0.7])), int(rng.integers(1 << 30)))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, k)]
        perm = rng.permutation(k)
        relab = [-1] * k
        for x in range(k):
            relab[perm[x]] = -1 if parent[x] < 0 else int(perm[parent[x]])
        col = rng.integers(0, k, n).astype(np.uint8)
        cases.append((g, relab, col))
    return cases


def test_small_suite_every_table_exact():
    for g, parent, col in _small_suite():
        got = tables(g, parent, col)
        ref = oracle_tables(g, parent, col, oracle.NUM_EXACT)
        for x in range(len(parent)):
            assert np.array_equal(got[x], ref[x]), (parent, x)


def test_more_colours_than_vertices_every_table_exact():
    """kc > k colours: every table, the root per-vertex counts and
    the total against the oracle's kc-colour DP (itself pinned to brute
    force), including heavy segments and fp32."""
    cc = lib()
    rng = np.random.default_rng(77)
    for trial in range(12):
        k = int(rng.integers(2, 8))
        kc = int(rng.integers(k + 1, min(k + 6, 16) + 1))
        n = int(rng.integers(k, 60))
        g = synth.gnp(n, float(rng.choice([0.1, 0.3])), int(rng.integers(1 << 30)))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, k)]
        col = rng.integers(0, kc, n).astype(np.uint8)
        want = oracle.dp_count(g, parent, col, oracle.NUM_EXACT, want_root=True, colours=kc)
        sizes = subtree_sizes(parent)
        with context(g, parent, segment_len=3) as ctx:
            cc.cc_set_template_colors(ctx, parent, kc)
            cc.cc_set_colors(ctx, col)
            assert cc.cc_count_colorful(ctx) == float(want.total), (k, kc, parent)
            root = cc.cc_get_subtree_counts(ctx, parent.index(-1), g.n, kc, kc)
            assert np.array_equal(root[:, 0], want.root), (k, kc)
            for x in range(k):
                if parent[x] < 0:
                    continue
                got = cc.cc_get_subtree_counts(ctx, x, g.n, kc, sizes[x])
                ref = oracle.dp_count(g, parent, col, oracle.NUM_EXACT, keep_x=x, colours=kc).table
                assert np.array_equal(got, ref), (k, kc, parent, x)
        with context(g, parent, "fp32") as ctx:
            cc.cc_set_template_colors(ctx, parent, kc)
            cc.cc_set_colors(ctx, col)
            assert rel_err(cc.cc_count_colorful(ctx), float(want.total)) <= TOL_FP32


def test_more_colours_estimator_scaling():
    """estimate = mean X_j kc^k (kc-k)! / kc! / |Aut(T)| for kc colours."""
    cc = lib()
    g = synth.gnp(40, 0.3, 3)
    parent = [-1, 0, 1, 1]
    k, kc = 4, 7
    with context(g, parent) as ctx:
        cc.cc_set_template_colors(ctx, parent, kc)
        est, xs = cc.cc_estimate(ctx, 12, 300, per_iter=True)
        est_m = cc.cc_estimate_mom(ctx, 12, 300, 3)
    want_x = [oracle.dp_count(g, parent, oracle.color(g.n, kc, 300 + j), oracle.NUM_EXACT, colours=kc).total
              for j in range(12)]
    assert list(xs) == [float(v) for v in want_x]
    scale = kc ** k * math.factorial(kc - k) / math.factorial(kc) / oracle.aut(parent)
    assert est == pytest.approx(np.mean(want_x) * scale, rel=1e-13)
    groups = [np.mean(want_x[0:4]), np.mean(want_x[4:8]), np.mean(want_x[8:12])]
    assert est_m == pytest.approx(float(np.median(groups)) * scale, rel=1e-13)


def test_multi_template_counts_share_tables():
    """cc_count_colorful_multi: several templates on one colouring,
    isomorphic sub-templates computed once -- every count equals the oracle's
    single-template DP, for kc = k and kc > k, fp64 and fp32."""
    cc = lib()
    templates = [[-1, 0, 1, 2, 3, 4], [-1, 0, 0, 0, 0, 0], [-1, 0, 1, 2, 3, 2], [-1, 0, 1, 2, 2, 2],
                 [-1, 0, 1, 1, 2, 2], [-1, 0, 0, 1, 1, 2], [-1, 0, 1], [-1, 0, 1, 2, 3, 4, 5, 6]]
    for gi, g in enumerate((synth.gnp(70, 0.12, 5), synth.scaled_twin(synth.CONFIGS[3], 11, 16).graph())):
        for kc in (8, 10):
            col = oracle.color(g.n, kc, 31 + gi)
            want = [oracle.dp_count(g, t, col, oracle.NUM_LONGDOUBLE, colours=kc).total for t in templates]
            with context(g, templates[0]) as ctx:
                cc.cc_set_template_colors(ctx, templates[0], kc)
                cc.cc_set_colors(ctx, col)
                got = cc.cc_count_colorful_multi(ctx, templates)
                reused = cc.cc_last_stats(ctx)["halo_bytes"]  # out[9]: tables reused across templates
                assert cc.cc_count_colorful(ctx) == got[0]  # the context's own template is restored
            for i, t in enumerate(templates):
                assert rel_err(got[i], want[i]) <= TOL_FP64, (gi, kc, t)
            assert reused > 0
            with context(g, templates[0], "fp32") as ctx:
                cc.cc_set_template_colors(ctx, templates[0], kc)
                cc.cc_set_colors(ctx, col)
                got32 = cc.cc_count_colorful_multi(ctx, templates)
            for i in range(len(templates)):
                assert rel_err(got32[i], want[i]) <= TOL_FP32


def test_small_suite_heavy_segments_and_chunks_do_not_change_results():
    for g, parent, col in _small_suite()[:10]:
        want = float(oracle.dp_count(g, parent, col, oracle.NUM_EXACT).total)
        for seg in (1, 2, 3):
            assert count(g, parent, colors=col, segment_len=seg) == want
        assert count(g, parent, colors=col, precision="fp32") == pytest.approx(want, rel=TOL_FP32)


# ------------------------------------------------------------------ fused root (root evaluated in the gather epilogue)
FUSED_CASES = [
    ([-1, 0, 0, 1, 1, 2, 2], 2),  # two identical subtrees under the root: self dot (mode 2)
    ([-1, 0, 1, 0, 3], 2),        # P5 rooted at its centre
    ([-1, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6], 2),  # configs[4]'s template
    ([-1, 0, 0, 2], 1),           # root with a leaf and a P2 child: dot with the active table (mode 1)
]


@pytest.mark.parametrize("parent,mode", FUSED_CASES)
def test_fused_root_exact(parent, mode):
    cc = lib()
    k = len(parent)
    graphs = [synth.gnp(60, 0.25, 11), synth.scaled_twin(synth.CONFIGS[3], 10, 16).graph()]
    for gi, g in enumerate(graphs):
        col = oracle.color(g.n, k, 40 + gi)
        want = oracle.dp_count(g, parent, col, oracle.NUM_EXACT, want_root=True)
        for seg in (0, 3):
            with context(g, parent, fixed_root=1, segment_len=seg) as ctx:
                cc.cc_set_colors(ctx, col)
                x = cc.cc_count_colorful(ctx)
                assert cc.cc_last_stats(ctx)["fused_root"] == mode
                root = cc.cc_get_subtree_counts(ctx, parent.index(-1), g.n, k, k)
                cc.cc_set_knob(ctx, "fused_root", 0)
                x_unfused = cc.cc_count_colorful(ctx)
                assert cc.cc_last_stats(ctx)["fused_root"] == 0
                cc.cc_set_knob(ctx, "fused_root", 1)
            # exact while every partial sum stays below 2^53; the 15-vertex tree's
            # root products do not, so the bar there is the fp64 1e-12
            assert rel_err(x, float(want.total)) <= TOL_FP64, (parent, gi, seg)
            assert rel_err(x_unfused, float(want.total)) <= TOL_FP64, (parent, gi, seg)
            assert_close_entries(root, want.root.reshape(-1, 1), TOL_FP64, f"fused root per vertex {parent}")
        with context(g, parent, "fp32", fixed_root=1) as ctx:
            cc.cc_set_colors(ctx, col)
            assert rel_err(cc.cc_count_colorful(ctx), float(want.total)) <= TOL_FP32


@pytest.mark.parametrize("ci", [2, 3])
def test_fused_combine_root(ci):
    """Fused combine + root (fused_root mode 3): configs[2]'s and [3]'s root
    step takes its active table from a register-blocked combine over the
    same passive neighbour sum, so X_v is formed in that combine's epilogue
    and the active table is never stored.  Against the oracle (count and
    every X_v) and the unfused run; fp64 where the Z-block kernel exists in
    fp64 (configs[2]'s (7;4,3)), fp32 for both."""
    cc = lib()
    cfg = synth.CONFIGS[ci]
    parent, k = cfg.parent, cfg.k
    graphs = [synth.gnp(70, 0.2, 5), synth.scaled_twin(cfg, 10, 16).graph()]
    precs = [("fp32", TOL_FP32)] + ([("fp64", TOL_FP64)] if ci == 2 else [])
    for gi, g in enumerate(graphs):
        col = oracle.color(g.n, k, 60 + gi)
        want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE, want_root=True)
        for prec, tol in precs:
            for seg in (0, 3):
                with context(g, parent, prec, segment_len=seg) as ctx:
                    cc.cc_set_colors(ctx, col)
                    x = cc.cc_count_colorful(ctx)
                    assert cc.cc_last_stats(ctx)["fused_root"] == 3, (ci, prec)
                    root = cc.cc_get_subtree_counts(ctx, parent.index(-1), g.n, k, k)
                    cc.cc_set_knob(ctx, "fused_root", 0)
                    x_unfused = cc.cc_count_colorful(ctx)
                    assert cc.cc_last_stats(ctx)["fused_root"] == 0
                    cc.cc_set_knob(ctx, "fused_root", 1)
                assert rel_err(x, float(want.total)) <= tol, (ci, gi, prec, seg)
                assert rel_err(x_unfused, x) <= tol
                assert_close_entries(root, want.root.reshape(-1, 1), tol, f"fused combine root X_v config {ci}")


@pytest.mark.parametrize("ci", [2, 3])
def test_static_cover_combine(ci):
    """The compile-time-cover combine (combine_s.cu, knob combine_static) for
    configs[2]'s (7;4,3) at k = 10 and configs[3]'s (9;6,3) at k = 12, fp32:
    fused with the root (T' never stored, X_v in its epilogue) and stored
    (fused_root = 0, the root step reads the table).  Count and every X_v
    against the oracle, and against the run-time-cover Z-block kernel
    (combine_static = 0), on a dense small graph, a twin with hubs and a
    ragged last tile (n not a multiple of 32)."""
    cc = lib()
    cfg = synth.CONFIGS[ci]
    parent, k = cfg.parent, cfg.k
    graphs = [synth.gnp(77, 0.2, 7), synth.scaled_twin(cfg, 10, 16).graph()]
    for gi, g in enumerate(graphs):
        col = oracle.color(g.n, k, 90 + gi)
        want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE, want_root=True)
        got = {}
        with context(g, parent, "fp32") as ctx:
            cc.cc_set_colors(ctx, col)
            for static in (2, 0):  # 2: the static kernel for both shapes
                cc.cc_set_knob(ctx, "combine_static", static)
                for fused in (1, 0):
                    cc.cc_set_knob(ctx, "fused_root", fused)
                    x = cc.cc_count_colorful(ctx)
                    assert cc.cc_last_stats(ctx)["fused_root"] == (3 if fused else 0), (ci, static, fused)
                    root = cc.cc_get_subtree_counts(ctx, parent.index(-1), g.n, k, k)
                    assert rel_err(x, float(want.total)) <= TOL_FP32, (ci, gi, static, fused)
                    assert_close_entries(root, want.root.reshape(-1, 1), TOL_FP32,
                                         f"static={static} fused={fused} X_v config {ci}")
                    got[static, fused] = x
        for key, x in got.items():
            assert rel_err(x, got[2, 1]) <= TOL_FP32, key


def test_subtree_rows_match_the_full_dump_and_the_oracle():
    """cc_get_subtree_rows (the sampled-row hook used at configs[4] scale)
    returns the same rows as the full-table dump and the oracle, including
    isolated vertices (zero rows) and the root column."""
    cc = lib()
    cfg = synth.scaled_twin(synth.CONFIGS[4], 10, 16)
    g0 = cfg.graph()
    g = synth.from_edges(g0.n + 3, np.stack(g0.edges(), axis=1))  # + 3 isolated vertices
    k = cfg.k
    col = oracle.color(g.n, k, 9)
    rng = np.random.default_rng(4)
    verts = np.concatenate([rng.choice(g0.n, 12, replace=False), [g.n - 1, g.n - 2]]).astype(np.int32)
    sizes = subtree_sizes(cfg.parent)
    with context(g, cfg.parent) as ctx:
        cc.cc_set_colors(ctx, col)
        got = {}
        for x in (1, 3, 7):  # B7, B3 and a leaf
            got[x] = rows = cc.cc_get_subtree_rows(ctx, x, verts, k, sizes[x])
            full = cc.cc_get_subtree_counts(ctx, x, g.n, k, sizes[x])
            assert np.array_equal(rows, full[verts]), x
            ref = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE, keep_x=x).table
            assert_close_entries(rows, ref[verts], TOL_FP64, f"rows x={x}")
        root = cc.cc_get_subtree_rows(ctx, 0, verts, k, k)
        want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE, want_root=True).root
        assert_close_entries(root[:, 0], want[verts], TOL_FP64, "root rows")
        assert np.all(got[1][-2:] == 0) and np.all(got[3][-2:] == 0)  # isolated: no tree of >= 2 vertices
        assert np.array_equal(got[7][-2:].sum(axis=1), [1.0, 1.0])  # ... but the single vertex maps


def test_sibling_pair_gather_every_row():
    """Sibling pairs (knob pair_gather = 1, one rank; off by default: measured
    slower): configs[3]'s plan sums the p = 2 passive (the lifted leaf level,
    11 columns) and B3 (the (3;2,1) combine, run ahead of its turn, 55
    columns) in ONE traversal of the colour-sorted lists (Eq. 1's inner sum,
    PAPER.md line 118, for both).  fp32 rows only: in fp64 the pair's rows
    (6 + 28 vectors) exceed the 24-vector limit and no pair forms.  Every
    full-subtree row of every template vertex is within the fp32 tolerance
    of the oracle, zero entries exactly zero; with forced heavy segments too
    (the segments' partial rows of both parts)."""
    cc = lib()
    cfg = synth.scaled_twin(synth.CONFIGS[3], 12, 32)
    g = cfg.graph()
    k = cfg.k
    col = oracle.color(g.n, k, 5)
    sizes = subtree_sizes(cfg.parent)
    verts = np.arange(g.n, dtype=np.int32)
    want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE, want_root=True)
    for seg in (0, 64):
        with context(g, cfg.parent, "fp64", segment_len=seg) as ctx:
            cc.cc_set_colors(ctx, col)
            cc.cc_set_knob(ctx, "pair_gather", 1)
            x64 = cc.cc_count_colorful(ctx)
            assert cc.cc_last_stats(ctx)["sibling_pairs"] == 0
            assert rel_err(x64, float(want.total)) <= TOL_FP64
        with context(g, cfg.parent, "fp32", segment_len=seg) as ctx:
            cc.cc_set_colors(ctx, col)
            cc.cc_set_knob(ctx, "pair_gather", 0)
            x0 = cc.cc_count_colorful(ctx)
            assert cc.cc_last_stats(ctx)["sibling_pairs"] == 0
            cc.cc_set_knob(ctx, "pair_gather", 1)
            x1 = cc.cc_count_colorful(ctx)
            assert cc.cc_last_stats(ctx)["sibling_pairs"] >= 1
            assert rel_err(x1, float(want.total)) <= TOL_FP32
            assert rel_err(x1, x0) <= TOL_FP32
            for x in range(k):
                if cfg.parent[x] == -1:
                    rows = cc.cc_get_subtree_rows(ctx, x, verts, k, k)[:, 0]
                    ref = want.root
                else:
                    rows = cc.cc_get_subtree_rows(ctx, x, verts, k, sizes[x])
                    ref = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE, keep_x=x).table
                assert_close_entries(rows, ref, TOL_FP32, f"pair x={x} seg={seg}")


# ------------------------------------------------------------------ configs[1]: fp64 1e-12 per entry, fp32 1e-4
def test_config1_fp64_every_entry_and_fp32_total():
    cfg = synth.CONFIGS[1]
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    ref = oracle_tables(g, cfg.parent, col, oracle.NUM_EXACT)
    got = tables(g, cfg.parent, col)
    for x in range(cfg.k):
        assert_close_entries(got[x], ref[x], TOL_FP64, f"config1 x={x}")
    want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_EXACT).total
    assert rel_err(count(g, cfg.parent, seed=cfg.color_seed), want) <= TOL_FP64
    assert rel_err(count(g, cfg.parent, seed=cfg.color_seed, precision="fp32"), want) <= TOL_FP32
    # heavy split forced (max degree ~9.6K) and narrow chunks: same result
    x1 = count(g, cfg.parent, seed=cfg.color_seed, segment_len=64)
    assert rel_err(x1, want) <= TOL_FP64


# ------------------------------------------------------------------ twins of configs 2-4 (oracle-sized)
@pytest.mark.parametrize("ci,scale,ef", [(2, 14, 16), (3, 13, 32), (4, 11, 64)])
def test_config_twins_fp64_every_entry(ci, scale, ef):
    cfg = synth.scaled_twin(synth.CONFIGS[ci], scale, ef)
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    ref = oracle_tables(g, cfg.parent, col, oracle.NUM_LONGDOUBLE)
    got = tables(g, cfg.parent, col, segment_len=256)
    for x in range(cfg.k):
        assert_close_entries(got[x], ref[x], TOL_FP64, f"{cfg.name} x={x}")


_SHORT_REF = {}


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_short_list_kernels_every_entry(prec, variant):
    """The short tail of the wide-row gathers (light items with <= 128
    neighbours; knob short_lists: 0 = with the long lists, 1 = k_gather_short,
    2-4 = the lean kernel at other occupancies) computes Eq. 1's neighbour sums
    (PAPER.md lines 114-120): every table of a configs[3] twin equals the
    oracle per entry (fp64 1e-12, fp32 1e-4; zero entries exactly zero),
    with heavy segments forced (s = 256) so both item kinds are present."""
    cc = lib()
    cfg = synth.scaled_twin(synth.CONFIGS[3], 13, 32)
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    if "ref" not in _SHORT_REF:
        _SHORT_REF["ref"] = oracle_tables(g, cfg.parent, col, oracle.NUM_LONGDOUBLE)
    ref = _SHORT_REF["ref"]
    sizes = subtree_sizes(cfg.parent)
    k = cfg.k
    tol = TOL_FP64 if prec == "fp64" else TOL_FP32
    with context(g, cfg.parent, prec, segment_len=256) as ctx:
        cc.cc_set_knob(ctx, "short_lists", variant)
        cc.cc_set_colors(ctx, col)
        for x in range(k):
            got = (cc.cc_get_subtree_counts(ctx, x, g.n, k, k) if cfg.parent[x] == -1
                   else cc.cc_get_subtree_counts(ctx, x, g.n, k, sizes[x]))
            assert_close_entries(got, ref[x], tol, f"short_lists={variant} {prec} x={x}")


@pytest.mark.parametrize("ci,scale,ef", [(2, 16, 16), (3, 14, 32), (4, 12, 64)])
def test_config_twins_fp32_total(ci, scale, ef):
    cfg = synth.scaled_twin(synth.CONFIGS[ci], scale, ef)
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE).total
    assert rel_err(count(g, cfg.parent, seed=cfg.color_seed, precision="fp32"), want) <= TOL_FP32
    assert rel_err(count(g, cfg.parent, seed=cfg.color_seed, precision="fp64"), want) <= TOL_FP64


# ------------------------------------------------------------------ configs[2] at full size
def test_config2_full_fp32_ten_colourings_one_and_two_ranks():
    """BASELINE.json configs[2] as specified: R-MAT scale 20, the 10-vertex
    spider, k = 10, fp32 tables with fp64 root, the 10 colourings of seeds
    2..11 (reading C-2), on one GPU and with the 1D partition over 2 ranks
    (loopback transport on this GPU; grouped exchange, whole-row and chunked
    halo rows): every X_j within 1e-4 of the oracle's fold-children DP."""
    from test_gpu_loopback import run_ranks
    cfg = synth.CONFIGS[2]
    g = cfg.graph()
    cc = lib()
    want = [float(oracle.dp_count(g, cfg.parent, oracle.color(g.n, cfg.k, cfg.color_seed + j), oracle.NUM_DOUBLE).total)
            for j in range(10)]
    with context(g, cfg.parent, "fp32") as ctx:
        _, xs = cc.cc_estimate(ctx, 10, cfg.color_seed, per_iter=True)
    for j in range(10):
        assert rel_err(xs[j], want[j]) <= TOL_FP32, (j, xs[j], want[j])
    for chunk in (0, 64):
        out, _ = run_ranks(g, cfg.parent, 2, precision="fp32", estimate=(10, cfg.color_seed), exchange=1,
                           chunk_cols=chunk)
        for r in range(2):
            est, xr = out[r]
            for j in range(10):
                assert rel_err(xr[j], want[j]) <= TOL_FP32, (chunk, r, j, xr[j], want[j])


def test_config3_full_size_fp32_vs_oracle():
    """configs[3] at full size (R-MAT scale 23, 507 M adjacency entries, the
    bench workload) against the oracle's fold-children DP in double on the
    host (~60 GB, a few minutes on 16 cores): final count within 1e-4."""
    cfg = synth.CONFIGS[3]
    g = cfg.graph()
    x = count(g, cfg.parent, seed=cfg.color_seed, precision="fp32")
    want = oracle.dp_count(g, cfg.parent, oracle.color(g.n, cfg.k, cfg.color_seed), oracle.NUM_DOUBLE).total
    assert rel_err(x, want) <= TOL_FP32


# ------------------------------------------------------------------ closed forms at any size
def test_star_closed_form_full_config3_graph():
    """X(star with k-1 leaves) = (k-1)! sum_v prod_{j != c_v} cnt_j(v) (SURVEY 8(c) pins)."""
    g = synth.CONFIGS[3].graph()
    k = 5
    col = oracle.color(g.n, k, 77)
    src = np.repeat(np.arange(g.n), g.degrees())
    lin = src.astype(np.int64) * k + col[g.col]
    cnt = np.bincount(lin, minlength=g.n * k).reshape(g.n, k).astype(np.float64)
    cnt[np.arange(g.n), col] = 1.0
    want = math.factorial(k - 1) * float(np.sum(np.prod(cnt, axis=1) * (g.degrees() > 0)))
    got = count(g, [-1] + [0] * (k - 1), seed=77, precision="fp64")
    assert rel_err(got, want) <= 1e-12


def test_clique_every_entry_closed_form():
    n = 300
    g = synth.clique(n)
    cfg = synth.CONFIGS[2]
    k = cfg.k
    col = oracle.color(n, k, 5)
    c = np.bincount(col, minlength=k).astype(np.float64)
    x = count(g, cfg.parent, colors=col)
    assert rel_err(x, math.factorial(k) * float(np.prod(c))) <= 1e-12
    got = tables(g, cfg.parent, col)
    sizes = subtree_sizes(cfg.parent)
    import itertools
    for xv in (1, 2):
        s = sizes[xv]
        subsets = sorted(itertools.combinations(range(k), s), key=lambda t: t[::-1])
        for v in (0, 7, 299):
            want = [math.factorial(s - 1) * math.prod(c[j] - (j == col[v]) for j in S if j != col[v])
                    if col[v] in S else 0.0 for S in subsets]
            assert_close_entries(got[xv][v], want, 1e-12, f"clique x={xv} v={v}")


def test_maximum_template_size_k16():
    """k = 16 (the library's maximum): P_16 on a long cycle with col = v mod 16
    (every window rainbow: X = 2n exactly), and a 16-vertex tree on an R-MAT
    graph against the oracle, fp64 per entry of the root counts."""
    n = 160_000
    assert count(synth.cycle(n), [-1] + list(range(15)), colors=(np.arange(n) % 16).astype(np.uint8)) == 2 * n
    parent = [-1] + [(i - 1) // 2 for i in range(1, 15)] + [14]  # binary tree of 15 plus a leaf under a leaf
    g = synth.rmat(9, 8, seed=3)
    col = oracle.color(g.n, 16, 5)
    want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE, want_root=True)
    for prec, tol in (("fp64", TOL_FP64), ("fp32", TOL_FP32)):
        with context(g, parent, prec) as ctx:
            cc = lib()
            cc.cc_set_colors(ctx, col)
            assert rel_err(cc.cc_count_colorful(ctx), want.total) <= tol
            if prec == "fp64":
                root = cc.cc_get_subtree_counts(ctx, 0, g.n, 16, 16)
                assert_close_entries(root[:, 0], want.root, TOL_FP64, "k=16 root")


def test_path_on_long_cycle():
    # P_k on C_n with col = v mod k, k | n: every window is rainbow, X = 2n (SURVEY 8(c) pins)
    n, k = 200_004, 6
    g = synth.cycle(n)
    col = (np.arange(n) % k).astype(np.uint8)
    assert count(g, [-1] + list(range(k - 1)), colors=col) == 2 * n
    # random colouring: X = 2 * #rainbow windows
    rng = np.random.default_rng(8)
    col = rng.integers(0, k, n).astype(np.uint8)
    win = np.ones(n, dtype=bool)
    for a in range(k):
        for b in range(a + 1, k):
            win &= col[(np.arange(n) + a) % n] != col[(np.arange(n) + b) % n]
    assert count(g, [-1] + list(range(k - 1)), colors=col, segment_len=1) == 2 * int(win.sum())


# ------------------------------------------------------------------ degenerate cases
def test_degenerate_cases():
    cc = lib()
    # k = 1: X = n (including isolated vertices)
    g = synth.from_edges(7, [(0, 1)])
    assert count(g, [-1], seed=1) == 7.0
    # k = 2: X = 2 * #bichromatic edges
    g = synth.rmat(10, 8, seed=4)
    col = oracle.color(g.n, 2, 3)
    eu, ev = g.edges()
    assert count(g, [-1, 0], colors=col) == 2 * int(np.sum(col[eu] != col[ev]))
    # n < k, edgeless, empty graph
    assert count(synth.path(3), [-1, 0, 1, 2], seed=1) == 0.0
    assert count(synth.from_edges(50, []), [-1, 0, 1], seed=1) == 0.0
    assert count(synth.from_edges(0, []), [-1, 0], seed=1) == 0.0
    # monochrome colouring
    assert count(synth.clique(6), [-1, 0, 1], colors=np.zeros(6, np.uint8)) == 0.0
    # G = T with a rainbow colouring: X = |Aut(T)|
    for cfg in synth.CONFIGS:
        gt = synth.tree_graph(cfg.parent)
        assert count(gt, cfg.parent, colors=np.arange(cfg.k, dtype=np.uint8)) == oracle.aut(cfg.parent)
    # k = 16 (maximum)
    par16 = [-1] + [(i - 1) // 2 for i in range(1, 16)]
    g16 = synth.tree_graph(par16)
    assert count(g16, par16, colors=np.arange(16, dtype=np.uint8)) == oracle.aut(par16)
    with context(synth.cycle(5), [-1, 0]) as ctx:
        aut, aut_root, ns = cc.cc_template_info(ctx)
        assert (aut, aut_root, ns) == (2, 1, 1)


def test_determinism_bitwise():
    cfg = synth.CONFIGS[1]
    g = cfg.graph()
    xs = {count(g, cfg.parent, seed=5, precision="fp32") for _ in range(3)}
    assert len(xs) == 1


def test_invariances():
    """SURVEY 8(c) invariants on the CUDA path, exact in fp64 (integer
    counts below 2^53): the count does not depend on the root and cut order
    (reading C-4: planner's choice vs the parent -1 vertex), on the internal
    vertex relabelling, on a permutation of the colour names, or on the
    heavy-vertex segment length; and equals the oracle's (exact below 2^53,
    else within the fp64 bar)."""
    rng = np.random.default_rng(8)
    cases = [(synth.scaled_twin(synth.CONFIGS[3], 10, 16).graph(), synth.CONFIGS[3].parent),
             (synth.scaled_twin(synth.CONFIGS[2], 10, 16).graph(), synth.CONFIGS[2].parent),
             (synth.gnp(120, 0.08, 6), [-1, 0, 1, 2, 2, 0, 5])]
    for g, parent in cases:
        k = len(parent)
        col = oracle.color(g.n, k, 77)
        want = float(oracle.dp_count(g, parent, col, oracle.NUM_EXACT).total)
        perm = rng.permutation(k).astype(np.uint8)
        runs = [count(g, parent, colors=col),
                count(g, parent, colors=col, fixed_root=1),
                count(g, parent, colors=col, relabel_seed=12345),
                count(g, parent, colors=perm[col]),
                count(g, parent, colors=col, segment_len=7)]
        # exact below 2^53; above it (the 12-vertex tree) within the fp64 bar
        assert all(rel_err(r, want) <= TOL_FP64 for r in runs), (parent, runs, want)
        if want < 2.0 ** 53:
            assert runs == [want] * len(runs), (parent, runs, want)


def test_estimator_matches_oracle_formula():
    cc = lib()
    g = synth.gnp(40, 0.3, 3)
    parent = [-1, 0, 1, 1]
    with context(g, parent) as ctx:
        est, xs = cc.cc_estimate(ctx, 50, 1000, per_iter=True)
    want_x = [oracle.dp_count(g, parent, oracle.color(g.n, 4, 1000 + j), oracle.NUM_EXACT).total for j in range(50)]
    assert list(xs) == [float(v) for v in want_x]
    assert est == pytest.approx(oracle.estimate(want_x, 4, oracle.aut(parent)), rel=1e-14)


def test_median_of_means_estimator_matches_oracle():
    cc = lib()
    g = synth.gnp(40, 0.3, 3)
    parent = [-1, 0, 1, 1]
    with context(g, parent) as ctx:
        est, xs = cc.cc_estimate_mom(ctx, 21, 500, 5, per_iter=True)
    want_x = [oracle.dp_count(g, parent, oracle.color(g.n, 4, 500 + j), oracle.NUM_EXACT).total for j in range(21)]
    assert list(xs) == [float(v) for v in want_x]
    assert est == pytest.approx(oracle.median_of_means(want_x, 4, oracle.aut(parent), 5), rel=1e-14)


# ------------------------------------------------------------------ errors
def test_errors_are_reported():
    cc = lib()
    ctx = cc.cc_create(device=0)
    try:
        with pytest.raises(cc.CCError) as e:
            cc.cc_count_colorful(ctx)
        assert e.value.status == cc.CC_ERR_STATE
        bad = synth.from_edges(3, [(0, 1)])
        col = bad.col.copy()
        col[0] = 2  # 0 -> 2 but 2 has no 0: asymmetric
        with pytest.raises(cc.CCError) as e:
            cc.cc_load_graph(ctx, 3, bad.row_ptr, col)
        assert e.value.status == cc.CC_ERR_GRAPH
        with pytest.raises(cc.CCError) as e:
            cc.cc_load_graph(ctx, 2, np.array([0, 1, 2]), np.array([0, 1], np.int32))  # self-loops
        assert e.value.status == cc.CC_ERR_GRAPH
        with pytest.raises(cc.CCError) as e:
            cc.cc_load_graph(ctx, 2, np.array([0, 2, 3]), np.array([1, 1, 0], np.int32))  # duplicate
        assert e.value.status == cc.CC_ERR_GRAPH
        for par in ([0, -1, 5], [-1, -1], [1, 0], list(range(-1, 16))):
            with pytest.raises(cc.CCError) as e:
                cc.cc_set_template(ctx, par)
            assert e.value.status == cc.CC_ERR_TEMPLATE
    finally:
        cc.cc_destroy(ctx)


def test_options_and_hooks_are_validated():
    cc = lib()
    with pytest.raises(cc.CCError) as e:
        cc.cc_create(device=0, chunk_cols=-1)  # >= 0
    assert e.value.status == cc.CC_ERR_ARG
    with pytest.raises(cc.CCError) as e:
        cc.cc_create(device=0, replicas=2)
    assert e.value.status == cc.CC_ERR_ARG
    with pytest.raises(cc.CCError) as e:
        cc.cc_create(device=0, exchange=5)  # CC_EXCHANGE_AUTO .. CC_EXCHANGE_DEVICE only
    assert e.value.status == cc.CC_ERR_ARG
    g = synth.gnp(50, 0.2, 1)
    with context(g, [-1, 0, 1, 2]) as ctx:  # P4: a p = 2 neighbour sum under every root
        with pytest.raises(cc.CCError) as e:
            cc.cc_set_template_colors(ctx, [-1, 0, 1, 2], 3)  # fewer colours than vertices
        assert e.value.status == cc.CC_ERR_ARG
        cc.cc_color(ctx, 3)
        x = cc.cc_count_colorful(ctx)
        cc.cc_set_profiling(ctx, False)
        assert cc.cc_count_colorful(ctx) == x
        prof = cc.cc_last_profile(ctx)
        assert prof["total"] > 0 and prof["gather"] == 0.0 and prof["csort"] == 0.0  # no per-kernel events
        cc.cc_set_profiling(ctx, True)
        assert cc.cc_count_colorful(ctx) == x
        prof = cc.cc_last_profile(ctx)
        assert prof["gather"] > 0 and prof["csort"] > 0
        with pytest.raises(cc.CCError) as e:
            cc.cc_set_colors(ctx, np.full(g.n, 7, np.uint8))  # colour out of range
        assert e.value.status == cc.CC_ERR_ARG


def test_fp32_overflow_is_reported_nonfinite():
    """Reading C-13: fp32 tables that overflow make the count non-finite and
    cc_count_colorful returns CC_ERR_NONFINITE.  A 16-vertex star on the
    clique K_2000 with 16 colours: the active table of the 15-vertex partial
    star holds 14! prod cnt_j ~ 2e40 > FLT_MAX; in fp64 the count is the
    clique closed form X = k! prod_j cnt_j (SURVEY 8(c) pins)."""
    cc = lib()
    n, k = 2000, 16
    g = synth.clique(n)
    parent = [-1] + [0] * (k - 1)
    col = oracle.color(n, k, 3)
    cnt = np.bincount(col, minlength=k).astype(np.float64)
    want = math.factorial(k) * float(np.prod(cnt))
    assert rel_err(count(g, parent, colors=col, precision="fp64"), want) <= TOL_FP64
    with context(g, parent, "fp32") as ctx:
        cc.cc_set_colors(ctx, col)
        with pytest.raises(cc.CCError) as e:
            cc.cc_count_colorful(ctx)
        assert e.value.status == cc.CC_ERR_NONFINITE
        # not poisoned: the context still counts (fp32 overflow is not a CUDA error)
        cc.cc_set_colors(ctx, np.zeros(n, np.uint8))
        assert cc.cc_count_colorful(ctx) == 0.0


KNOB_SETTINGS = [("gather_impl", 1), ("gather_impl", 2), ("narrow_impl", 0), ("narrow_impl", 1),
                 ("narrow_split", 0), ("narrow_split", 7), ("csort_small", 0), ("sector_skip", 0),
                 ("combine_impl", 1), ("combine_impl", 2), ("combine_impl", 3), ("combine_impl", 4), ("acc32", 0),
                 ("fused_root", 0), ("phase_events", 0), ("hub_l2_pct", 0), ("grid_reserve", 32), ("layout", 1), ("short_lists", 0), ("short_lists", 1), ("short_lists", 3), ("short_split", 1), ("lean_split", 2),
                 ("pair_gather", 1), ("rows_variant", 2), ("short_lists", 4), ("combine_wreg", 0),
                 ("combine_static", 0), ("combine_static", 2), ("combine_zglobal", 0), ("tail_warps", 8), ("tail_warps", 2)]


@pytest.mark.parametrize("ci", [2, 3, 4])
def test_every_knob_setting_computes_the_same_count(ci):
    """The implementation knobs select kernels, never results:
    fp64 counts equal the oracle within 1e-12 under every setting (exactly
    equal to the default when the integer counts stay below 2^53), fp32
    within 1e-4."""
    cc = lib()
    cfg = synth.scaled_twin(synth.CONFIGS[ci], 11, 16)
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, 23)
    want = float(oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE).total)
    for prec, tol in (("fp64", TOL_FP64), ("fp32", TOL_FP32)):
        with context(g, cfg.parent, prec, segment_len=64) as ctx:
            cc.cc_set_colors(ctx, col)
            base = cc.cc_count_colorful(ctx)
            assert rel_err(base, want) <= tol
            for name, value in KNOB_SETTINGS:
                old = cc.cc_get_knob(ctx, name)
                cc.cc_set_knob(ctx, name, value)
                x = cc.cc_count_colorful(ctx)
                cc.cc_set_knob(ctx, name, old)
                assert rel_err(x, want) <= tol, (ci, prec, name, value, x, want)
                if prec == "fp64" and want < 2.0 ** 53:
                    assert x == base, (ci, name, value)
        with pytest.raises(cc.CCError) as e:
            with context(g, cfg.parent) as ctx:
                cc.cc_set_knob(ctx, "no_such_knob", 1)
        assert e.value.status == cc.CC_ERR_ARG


def test_cuda_graph_replay_equals_direct_counts():
    """use_graphs = 1 (configs[0] and [1], the launch-bound ones): the count's
    device work is captured once and replayed for every new colouring (data
    only); a knob change or a new template recaptures.  Every count equals
    the direct path's, which equals the oracle (fp64 exact)."""
    cc = lib()
    for ci in (0, 1):
        cfg = synth.CONFIGS[ci]
        g = cfg.graph()
        with context(g, cfg.parent) as direct, context(g, cfg.parent, use_graphs=1) as graphed:
            for seed in (2, 3, 4):
                cc.cc_color(direct, seed)
                cc.cc_color(graphed, seed)
                x = cc.cc_count_colorful(direct)
                assert cc.cc_count_colorful(graphed) == x, (ci, seed)
                assert cc.cc_last_profile(graphed)["total"] > 0
            want = oracle.dp_count(g, cfg.parent, oracle.color(g.n, cfg.k, 4), oracle.NUM_EXACT).total
            assert rel_err(x, float(want)) <= TOL_FP64  # (configs[1]'s counts pass 2^53)
            cc.cc_set_knob(graphed, "gather_impl", 2)  # recapture
            assert cc.cc_count_colorful(graphed) == x
            cc.cc_set_template(graphed, [-1, 0, 1])    # new plan: recapture
            cc.cc_set_template(direct, [-1, 0, 1])
            cc.cc_color(direct, 9)
            cc.cc_color(graphed, 9)
            assert cc.cc_count_colorful(graphed) == cc.cc_count_colorful(direct)
            e1, xs1 = cc.cc_estimate(graphed, 4, 50, per_iter=True)
            e2, xs2 = cc.cc_estimate(direct, 4, 50, per_iter=True)
            assert list(xs1) == list(xs2) and e1 == e2
