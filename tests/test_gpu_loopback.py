"""-m gpu: the multi-rank device path (1D vertex partition, Alg. 2 of the
paper; and colouring replicas) with several ranks on
ONE GPU through the in-process loopback transport (cc_options.loopback): each
rank is a host thread with its own context and partition; halo rows move by
event-ordered device copies and the final reductions on the host, so no
kernel waits for another rank.  Everything but NCCL itself runs: the
partition, the per-rank colour sort of the local / remote neighbour ranges,
the leaf level over the full ranges, the pack kernel, the halo placement, the
local gather and the accumulating remote gather, and the cross-rank sums.
The results must equal the single-rank run and the oracle."""
import threading

import numpy as np
import pytest

import oracle
import synth
from gpu_util import count, lib, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def run_ranks(g, parent, world, colors=None, seed=None, precision="fp64", replicas=0, estimate=None, **kw):
    cc = lib()
    group = cc.cc_loopback_create(world)
    out = [None] * world
    stats = [None] * world
    errors = []

    def worker(r):
        ctx = None
        try:
            opt = cc.cc_default_options(world=world, rank=r, device=0, replicas=replicas,
                                        precision=cc.CC_FP64 if precision == "fp64" else cc.CC_FP32, **kw)
            opt.loopback = group
            ctx = cc.cc_create(opt)
            cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
            cc.cc_set_template(ctx, parent)
            if estimate:
                out[r] = cc.cc_estimate(ctx, estimate[0], estimate[1], per_iter=True)
            else:
                if colors is not None:
                    cc.cc_set_colors(ctx, colors)
                else:
                    cc.cc_color(ctx, seed)
                out[r] = cc.cc_count_colorful(ctx)
                stats[r] = cc.cc_last_stats(ctx)
        except Exception as e:  # noqa: BLE001
            errors.append((r, e))
        finally:
            if ctx is not None:
                cc.cc_destroy(ctx)

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=900)
    cc.cc_loopback_destroy(group)
    assert not errors, errors
    return out, stats


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partitioned_counts_equal_single_rank_exact(world):
    rng = np.random.default_rng(world)
    cases = [(synth.CONFIGS[0].graph(), synth.CONFIGS[0].parent, 5),
             (synth.gnp(300, 0.05, 9), [-1, 0, 1, 1, 0, 4], 6),
             (synth.scaled_twin(synth.CONFIGS[3], 11, 16).graph(), synth.CONFIGS[3].parent, 12)]
    for g, parent, k in cases:
        col = rng.integers(0, k, g.n).astype(np.uint8)
        want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE).total
        single = count(g, parent, colors=col)
        for seg in (0, 3):
            xs, st = run_ranks(g, parent, world, colors=col, segment_len=seg)
            assert len(set(xs)) == 1, xs  # every rank returns the all-reduced count
            assert rel_err(xs[0], want) <= 1e-12 and rel_err(xs[0], single) <= 1e-12, (world, k, seg)
            if g.nnz > 1000:
                assert all(s["halo_bytes"] > 0 for s in st)  # rows really crossed between ranks


def test_partitioned_fp32_config1_and_twin_of_config4():
    for cfg, g in ((synth.CONFIGS[1], synth.CONFIGS[1].graph()),
                   (synth.CONFIGS[4], synth.scaled_twin(synth.CONFIGS[4], 11, 32).graph())):
        col = oracle.color(g.n, cfg.k, cfg.color_seed)
        want = oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE).total
        xs, _ = run_ranks(g, cfg.parent, 2, seed=cfg.color_seed, precision="fp32")
        assert rel_err(xs[0], want) <= 1e-4 and len(set(xs)) == 1
        xs, _ = run_ranks(g, cfg.parent, 2, seed=cfg.color_seed, precision="fp64")
        assert rel_err(xs[0], want) <= 1e-12


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_fused_root(world):
    """The fused root (reading C-15) in the partitioned path: the halo rows of
    the root's passive table arrive first and the full neighbour ranges are
    colour-sorted, so configs[4]'s N7 never reaches HBM on any rank (what
    lets configs[4] fit at P = 2).  Self dot (mode 2) and dot with the active
    table (mode 1), heavy segments, fp64 and fp32."""
    cases = [(synth.scaled_twin(synth.CONFIGS[4], 11, 32).graph(), synth.CONFIGS[4].parent, 2),
             (synth.gnp(200, 0.06, 8), [-1, 0, 0, 2], 1),
             (synth.gnp(200, 0.06, 9), [-1, 0, 0, 1, 1, 2, 2], 2)]
    for g, parent, mode in cases:
        k = len(parent)
        col = oracle.color(g.n, k, 12)
        want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE).total
        for prec, tol in (("fp64", 1e-12), ("fp32", 1e-4)):
            xs, st = run_ranks(g, parent, world, colors=col, precision=prec, segment_len=5, fixed_root=1)
            assert len(set(xs)) == 1 and rel_err(xs[0], want) <= tol, (parent, prec)
            assert all(s["fused_root"] == mode for s in st)


def test_colouring_replicas_split_the_iterations():
    """Replicas: every rank the whole graph, iteration j on rank
    j mod world, one all-reduce of the per-iteration counts."""
    g = synth.gnp(80, 0.1, 4)
    parent = [-1, 0, 1, 1]
    want_x = [oracle.dp_count(g, parent, oracle.color(g.n, 4, 70 + j), oracle.NUM_EXACT).total for j in range(9)]
    out, _ = run_ranks(g, parent, 3, replicas=1, estimate=(9, 70))
    for est, xs in out:
        assert list(xs) == [float(v) for v in want_x]
        assert est == pytest.approx(oracle.estimate(want_x, 4, oracle.aut(parent)), rel=1e-14)


def test_partitioned_config3_full_size_two_ranks():
    """configs[3] at full size split over 2 ranks (loopback, one GPU): the
    same count as the single-rank run (fp32 tables, different summation
    order: within 1e-6), with ~40% of the rows crossing as halos."""
    cfg = synth.CONFIGS[3]
    g = cfg.graph()
    single = count(g, cfg.parent, seed=cfg.color_seed, precision="fp32")
    xs, st = run_ranks(g, cfg.parent, 2, seed=cfg.color_seed, precision="fp32")
    assert len(set(xs)) == 1
    assert rel_err(xs[0], single) <= 1e-6
    assert all(s["halo_bytes"] > 0 for s in st)


@pytest.mark.parametrize("world", [3, 4])
def test_ring_and_grouped_exchange_schedules_agree(world):
    """SURVEY F2 / PAPER.md Alg. 3: the ring pipeline (step r sends to rank +
    r, receives from rank - r, the remote pass over that peer's rows while the
    next step transfers) and the grouped all-to-all give the oracle's count on
    every rank; the schedule in use is reported; auto picks the same one on
    every rank.  Heavy segments (segment_len 3) inside the per-peer passes,
    the fused root (whole ranges after the last step), fp64 and fp32."""
    cases = [(synth.scaled_twin(synth.CONFIGS[3], 11, 16).graph(), synth.CONFIGS[3].parent),
             (synth.scaled_twin(synth.CONFIGS[4], 11, 32).graph(), synth.CONFIGS[4].parent),
             (synth.gnp(300, 0.05, 9), [-1, 0, 1, 1, 0, 4])]
    for g, parent in cases:
        k = len(parent)
        col = oracle.color(g.n, k, 21)
        want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE).total
        for mode in (lib().CC_EXCHANGE_GROUPED, lib().CC_EXCHANGE_RING):
            for prec, tol, seg in (("fp64", 1e-12, 3), ("fp32", 1e-4, 0)):
                xs, st = run_ranks(g, parent, world, colors=col, precision=prec, segment_len=seg, exchange=mode)
                assert len(set(xs)) == 1 and rel_err(xs[0], want) <= tol, (parent, mode, prec)
                assert all(s["exchange"] == mode for s in st)
        xs, st = run_ranks(g, parent, world, colors=col)
        assert rel_err(xs[0], want) <= 1e-12
        assert len({s["exchange"] for s in st}) == 1 and st[0]["exchange"] in (1, 2)


def test_nccl_calls_on_one_rank():
    """The NCCL half of the partitioned path that one GPU can run: the
    library loads NCCL at run time, builds a communicator and moves fp64
    values with the same grouped ncclSend/ncclRecv and ncclAllReduce calls
    (and argument types) the halo exchange and the final reduction use."""
    lib().cc_nccl_selftest(0)


def test_ranks_plan_from_the_global_degree():
    """Every rank must run the SAME plan (the exchanges of different plans do
    not match).  The planner's root depends on the average degree; this
    template's choice switches inside the spread of the per-rank averages of
    an 8-way split of R-MAT scale 13, so a per-rank statistic
    would diverge.  With the global statistic the 8 ranks agree with the
    single-rank count and the oracle."""
    cc = lib()
    parent = [-1, 0, 0, 2, 0, 0, 1, 3, 6, 6, 0, 5]
    roots = {cc.cc_plan_template_auto(parent, d, 8)["root"] for d in (28.0, 32.0, 36.0, 40.0)}
    assert len(roots) > 1, "the template's plan must switch inside the per-rank degree spread"
    g = synth.rmat(13, 16, seed=5)
    k = len(parent)
    col = oracle.color(g.n, k, 17)
    want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE).total
    one = count(g, parent, colors=col)
    assert rel_err(one, want) <= 1e-12
    for world in (4, 8):
        got, _ = run_ranks(g, parent, world, colors=col)
        assert all(x == got[0] for x in got)
        assert rel_err(got[0], want) <= 1e-12, (world, got[0], want)


@pytest.mark.parametrize("world,exchange", [(2, 1), (3, 1), (3, 2), (4, 2), (3, 3)])
def test_chunked_exchange_equals_the_oracle(world, exchange):
    """chunk_cols > 0 with the 1D partition: per column chunk the boundary
    rows are packed, exchanged into one of two chunk-wide halo buffers and
    summed by the remote passes while the next chunk transfers; tables keep
    owned rows only.  Grouped (1) and ring (2) schedules, fp64 exact against
    the oracle, fp32 within 1e-4, ragged chunks (24 columns)."""
    rng = np.random.default_rng(10 + world)
    cases = [(synth.scaled_twin(synth.CONFIGS[3], 11, 16).graph(), synth.CONFIGS[3].parent),
             (synth.scaled_twin(synth.CONFIGS[4], 10, 32).graph(), synth.CONFIGS[4].parent),
             (synth.gnp(200, 0.06, 4), [-1, 0, 1, 1, 0, 4, 5])]
    for ci, (g, parent) in enumerate(cases):
        k = len(parent)
        col = rng.integers(0, k, g.n).astype(np.uint8)
        want = oracle.dp_count(g, parent, col, oracle.NUM_LONGDOUBLE).total
        for w in (24, 64):
            got, stats = run_ranks(g, parent, world, colors=col, chunk_cols=w, exchange=exchange, segment_len=64)
            assert all(x == got[0] for x in got)
            assert rel_err(got[0], want) <= 1e-12, (world, exchange, w, parent)
            assert stats[0]["exchange"] == exchange
            assert stats[0]["column_chunks"] > 0 or ci == 2  # (the k = 7 rows have <= 20 columns)
        got32, _ = run_ranks(g, parent, world, colors=col, precision="fp32", chunk_cols=64, exchange=exchange)
        assert rel_err(got32[0], want) <= 1e-4
