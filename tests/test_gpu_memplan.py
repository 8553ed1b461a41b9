"""-m gpu: the memory plan ("intermediate
data partitioning", lines 391-396 and 420-428 PeakMem): column chunks of the
neighbour sums (cc_options.chunk_cols), the row-batched tail of the plan and
the per-batch recomputation of the tail's passive table in column chunks.
Every variant is an exact regrouping of the same sums, so fp64 results equal
the oracle within the 1e-12 bar (exactly while the counts stay below 2^53)
and fp32 within 1e-4."""
import math

import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_close_entries, context, count, lib, rel_err

pytestmark = pytest.mark.gpu

TOL_FP64 = 1e-12
TOL_FP32 = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


TWINS = [(1, 16, 16), (2, 13, 16), (3, 12, 32), (4, 11, 64)]


@pytest.mark.parametrize("ci,scale,ef", TWINS)
def test_column_chunks_equal_the_oracle(ci, scale, ef):
    """chunk_cols > 0: every neighbour sum runs as one launch per chunk of
    its passive columns, the later ones accumulating into N''.  Widths that
    leave a ragged last chunk, one column group, and wider than any row."""
    cc = lib()
    cfg = synth.scaled_twin(synth.CONFIGS[ci], scale, ef) if ci > 1 else synth.CONFIGS[1]
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, 31)
    want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE, want_root=True)
    base = count(g, cfg.parent, colors=col)
    for w in (8, 24, 64, 4096):
        with context(g, cfg.parent, chunk_cols=w, segment_len=64) as ctx:
            cc.cc_set_colors(ctx, col)
            x = cc.cc_count_colorful(ctx)
            st = cc.cc_last_stats(ctx)
            root = cc.cc_get_subtree_counts(ctx, cfg.parent.index(-1), g.n, cfg.k, cfg.k)
        assert rel_err(x, float(want.total)) <= TOL_FP64, (ci, w)
        if float(want.total) < 2.0 ** 53:
            assert x == base
        assert_close_entries(root[:, 0], want.root, TOL_FP64, f"chunked root X_v ci={ci} w={w}")
        if w < 64 and ci > 1:  # (configs[1]'s passive rows have <= 15 columns)
            assert st["column_chunks"] > 0
        x32 = count(g, cfg.parent, colors=col, precision="fp32", chunk_cols=w)
        assert rel_err(x32, float(want.total)) <= TOL_FP32, (ci, w)


@pytest.mark.parametrize("ci,scale,ef", TWINS)
def test_row_batched_tail_equals_the_oracle(ci, scale, ef):
    """The memory plan's row-batched tail, forced by knobs: the last neighbour
    sum and the steps after it run per batch of rows (2, 5 batches), with the
    tail's passive table stored, or recomputed per batch in column chunks
    (8, 40 columns) by its combine when the plan allows it.  Count and every
    X_v against the oracle; fused root modes are replaced by the batch root."""
    cc = lib()
    cfg = synth.scaled_twin(synth.CONFIGS[ci], scale, ef) if ci > 1 else synth.CONFIGS[1]
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, 37)
    want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE, want_root=True)
    r = cfg.parent.index(-1)
    for prec, tol in (("fp64", TOL_FP64), ("fp32", TOL_FP32)):
        for nb, rcw in ((2, 0), (5, 0), (2, 8), (5, 40)):
            with context(g, cfg.parent, prec, segment_len=64) as ctx:
                cc.cc_set_colors(ctx, col)
                cc.cc_set_knob(ctx, "tail_batches", nb)
                cc.cc_set_knob(ctx, "tail_recompute_cols", rcw)
                x = cc.cc_count_colorful(ctx)
                st = cc.cc_last_stats(ctx)
                assert st["tail_batches"] == nb, (ci, st)
                root = cc.cc_get_subtree_counts(ctx, r, g.n, cfg.k, cfg.k)
            assert rel_err(x, float(want.total)) <= tol, (ci, prec, nb, rcw, x, float(want.total))
            assert_close_entries(root[:, 0], want.root, tol if prec == "fp64" else 1e-4,
                                 f"batched root X_v ci={ci} {prec} nb={nb} rc={rcw}")


def test_row_batched_tail_small_suite_exact():
    """Random trees on random graphs, heavy segments (s = 3) and the forced
    tail batches with recomputation: exact counts (integers < 2^53)."""
    cc = lib()
    rng = np.random.default_rng(99)
    for trial in range(24):
        k = int(rng.integers(3, 10))
        n = int(rng.integers(k, 80))
        g = synth.gnp(n, float(rng.choice([0.1, 0.3])), int(rng.integers(1 << 30)))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, k)]
        col = rng.integers(0, k, n).astype(np.uint8)
        want = float(oracle.dp_count(g, parent, col, oracle.NUM_EXACT).total)
        for nb, rcw, chunk in ((3, 0, 0), (4, 8, 0), (2, 16, 8)):
            with context(g, parent, segment_len=3, chunk_cols=chunk) as ctx:
                cc.cc_set_colors(ctx, col)
                cc.cc_set_knob(ctx, "tail_batches", nb)
                cc.cc_set_knob(ctx, "tail_recompute_cols", rcw)
                assert cc.cc_count_colorful(ctx) == want, (parent, nb, rcw, chunk)


def test_config3_full_size_chunk64_equals_unchunked():
    """configs[3] at full size with chunk_cols = 64 (the p = 5 passive's 330
    columns in 6 launches, p = 4's 165 in 3, ...) gives the unchunked count:
    fp32 tables, the only difference is where the fp32 block sums are cut."""
    cfg = synth.CONFIGS[3]
    g = cfg.graph()
    a = count(g, cfg.parent, seed=cfg.color_seed, precision="fp32")
    b = count(g, cfg.parent, seed=cfg.color_seed, precision="fp32", chunk_cols=64)
    assert rel_err(b, a) <= 1e-6, (a, b)


def test_memory_plan_batches_only_when_needed():
    """The automatic memory plan leaves a plan that fits alone (configs[2]:
    no batches, the fused root runs) and never changes the count."""
    cc = lib()
    cfg = synth.CONFIGS[2]
    g = cfg.graph()
    with context(g, cfg.parent, "fp32") as ctx:
        cc.cc_color(ctx, cfg.color_seed)
        x = cc.cc_count_colorful(ctx)
        st = cc.cc_last_stats(ctx)
        assert st["tail_batches"] == 0 and st["fused_root"] == 3
        cc.cc_set_knob(ctx, "tail_batches", 3)
        assert rel_err(cc.cc_count_colorful(ctx), x) <= 1e-6
