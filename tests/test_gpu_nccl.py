"""-m gpu, >= 2 GPUs: the 1D vertex partition over REAL NCCL (one process per
GPU, Alg. 2, the ring of Alg. 3 lines 279-324 and the
pipeline of lines 326-341), against the oracle.  Skipped when fewer than two
CUDA devices are visible (the loopback tests cover the device path on one
GPU; nothing here runs two ranks on one GPU).

Each rank process binds its GPU, joins a gloo group only to broadcast the
NCCL unique id (cc.distributed_options), and runs the library with world > 1:
colour sort of the local / remote ranges, pack kernel, grouped or ring
ncclSend/ncclRecv on the comm stream, remote passes, ncclAllReduce of the
count.  Every rank must return the oracle's count (fp64 1e-12, fp32 1e-4).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL_FP64 = 1e-12
TOL_FP32 = 1e-4


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    # name: (graph builder, parent, precision, iterations, seed0)
    "config2": (lambda: synth.CONFIGS[2].graph(), synth.CONFIGS[2].parent, "fp32", 10, 2),
    "twin3_fp64": (lambda: synth.scaled_twin(synth.CONFIGS[3], 13, 32).graph(), synth.CONFIGS[3].parent, "fp64", 2, 7),
    "twin4_fp64": (lambda: synth.scaled_twin(synth.CONFIGS[4], 11, 64).graph(), synth.CONFIGS[4].parent, "fp64", 2, 7),
    "twin4_fp32": (lambda: synth.scaled_twin(synth.CONFIGS[4], 12, 64).graph(), synth.CONFIGS[4].parent, "fp32", 2, 9),
}


def _rank(rank, world, port, case, exchange, chunk_cols, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                          LOCAL_RANK=str(rank))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1804_09764_b200 as cc
        build, parent, prec, iters, seed0 = CASES[case]
        g = build()
        opt, _buf = cc.distributed_options(precision=cc.CC_FP64 if prec == "fp64" else cc.CC_FP32,
                                           exchange=exchange, chunk_cols=chunk_cols, segment_len=256)
        ctx = cc.cc_create(opt)
        try:
            cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
            cc.cc_set_template(ctx, parent)
            _, xs = cc.cc_estimate(ctx, iters, seed0, per_iter=True)
            st = cc.cc_last_stats(ctx)
        finally:
            cc.cc_destroy(ctx)
        q.put((rank, list(map(float, xs)), st["exchange"], st["halo_bytes"]))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None, None))


def _run(world, case, exchange, chunk_cols=0):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, case, exchange, chunk_cols, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=1800) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errors = [o for o in out if not isinstance(o[1], list)]
    assert not errors, errors
    return sorted(out)


_want_cache = {}


def _want(case):
    if case not in _want_cache:
        build, parent, prec, iters, seed0 = CASES[case]
        g = build()
        num = oracle.NUM_DOUBLE if prec == "fp32" else oracle.NUM_LONGDOUBLE
        _want_cache[case] = [float(oracle.dp_count(g, parent, oracle.color(g.n, len(parent), seed0 + j), num).total)
                             for j in range(iters)]
    return _want_cache[case]


def _worlds():
    n = _ngpus()
    return sorted({w for w in (2, min(n, 4), min(n, 8)) if 2 <= w <= n})


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 CUDA devices (one rank per GPU)")
@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("exchange", [1, 2, 3, 4])  # grouped, ring, ncclAlltoAll, device-initiated stores
def test_nccl_partitioned_counts_equal_the_oracle(case, exchange):
    want = _want(case)
    tol = TOL_FP64 if CASES[case][2] == "fp64" else TOL_FP32
    for world in _worlds():
        for chunk in (0, 96):
            out = _run(world, case, exchange, chunk)
            for rank, xs, xmode, halo in out:
                assert xmode == exchange, (rank, xmode)
                assert halo > 0
                for j, (x, w) in enumerate(zip(xs, want)):
                    assert abs(x - w) <= tol * abs(w), (case, world, exchange, chunk, rank, j, x, w)
            assert all(o[1] == out[0][1] for o in out), "ranks disagree"


def test_nccl_device_api_one_rank_selftest():
    """The device-initiated exchange's machinery (NCCL >= 2.28 device API) on a
    one-rank communicator: symmetric window, device communicator with LSA
    barriers, stores through ncclGetLsaPointer, barrier, read back.  Runs on
    one GPU (no second rank is emulated)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_09764_b200 as cc
    cc.cc_nccl_device_selftest(0)
    cc.cc_nccl_selftest(0)
