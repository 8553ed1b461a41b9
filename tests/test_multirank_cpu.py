"""-m "not gpu": the N > 1 host path on CPU with gloo (world 2 grouped, world 3 ring).

Each rank takes its 1D-partition plan from the product library
(`cc_partition_plan`, the same host code `cc_load_graph` runs), exchanges the
boundary rows of a passive table with its peer exactly as the plan says (send
lists in the peer's receive order), aggregates over its local CSR, and checks
the result against the single-process neighbour sum.  This is the exchange
protocol of Alg. 2 that the NCCL path implements.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, scale, W, errq, schedule="grouped"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import torch

        import paper_1804_09764_b200 as cc
        g = synth.rmat(scale, 8, seed=5)
        P = np.random.default_rng(1).random((g.n, W))  # a passive table, rows by original id
        plan = cc.cc_partition_plan(g.n, g.row_ptr, g.col, world, rank)
        n_own = len(plan["own_orig"])
        n_halo = len(plan["halo_orig"])
        local = np.zeros((n_own + n_halo, W))
        local[:n_own] = P[plan["own_orig"]]
        rp, col = plan["rp"], plan["col"]
        if schedule == "ring":
            # Alg. 3 ring (CC_EXCHANGE_RING): step r sends to rank + r and
            # receives from rank - r; the remote sum over that peer's rows
            # (each row's halo range split at the peer's recv_off boundary)
            # accumulates as soon as they are in
            N = np.zeros((n_own, W))
            for i in range(n_own):
                nb = col[rp[i]:rp[i + 1]]
                nb = nb[nb < n_own]
                N[i] = local[nb].sum(axis=0)
            for r in range(1, world):
                dst, src = (rank + r) % world, (rank - r) % world
                s0, s1 = plan["send_off"][dst], plan["send_off"][dst + 1]
                req = dist.isend(torch.from_numpy(np.ascontiguousarray(local[plan["send_idx"][s0:s1]])), dst)
                r0, r1 = plan["recv_off"][src], plan["recv_off"][src + 1]
                buf = torch.zeros((r1 - r0, W), dtype=torch.float64)
                dist.recv(buf, src)
                req.wait()
                local[n_own + r0:n_own + r1] = buf.numpy()
                for i in range(n_own):
                    nb = col[rp[i]:rp[i + 1]]
                    lo = np.searchsorted(nb, n_own + r0)
                    hi = np.searchsorted(nb, n_own + r1)
                    N[i] += local[nb[lo:hi]].sum(axis=0)
            src_ = np.repeat(np.arange(g.n), g.degrees())
            NG = np.zeros((g.n, W))
            np.add.at(NG, src_, P[g.col])
            assert np.allclose(N, NG[plan["own_orig"]], rtol=1e-12, atol=0)
        # grouped send/recv with every peer (the NCCL step)
        reqs = []
        for q in range(world):
            if q == rank:
                continue
            s0, s1 = plan["send_off"][q], plan["send_off"][q + 1]
            send = torch.from_numpy(np.ascontiguousarray(local[plan["send_idx"][s0:s1]]))
            reqs.append(dist.isend(send, q))
        for q in range(world):
            if q == rank:
                continue
            r0, r1 = plan["recv_off"][q], plan["recv_off"][q + 1]
            buf = torch.zeros((r1 - r0, W), dtype=torch.float64)
            dist.recv(buf, q)
            local[n_own + r0:n_own + r1] = buf.numpy()
        for r in reqs:
            r.wait()
        # the halo rows are the rows of the global table
        assert np.array_equal(local[n_own:], P[plan["halo_orig"]])
        # local aggregation == global aggregation on owned rows
        rp, col = plan["rp"], plan["col"]
        N_local = np.add.reduceat(local[col], rp[:-1], axis=0) if len(col) else np.zeros((n_own, W))
        N_local[np.diff(rp) == 0] = 0
        src = np.repeat(np.arange(g.n), g.degrees())
        N_global = np.zeros((g.n, W))
        np.add.at(N_global, src, P[g.col])
        assert np.allclose(N_local, N_global[plan["own_orig"]], rtol=1e-12, atol=0)
        # every rank derived the same partition: owned sets are disjoint and cover
        owned = [None] * world
        dist.all_gather_object(owned, plan["own_orig"].tolist())
        allv = sorted(v for o in owned for v in o)
        assert allv == sorted(np.nonzero(g.degrees())[0].tolist())
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("world,schedule", [(2, "grouped"), (3, "ring")])
def test_halo_exchange_gloo(world, schedule):
    import __graft_entry__
    __graft_entry__._product_build()
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 11, 6, errq, schedule)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def _opts_worker(rank, world, port, errq, outq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        os.environ["LOCAL_RANK"] = str(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import ctypes

        import paper_1804_09764_b200 as cc
        opt, buf = cc.distributed_options(precision=cc.CC_FP32, exchange=cc.CC_EXCHANGE_RING)
        uid = ctypes.string_at(opt.nccl_id, 128)
        outq.put((rank, opt.world, opt.rank, opt.device, opt.precision, opt.exchange, uid))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def test_distributed_options_share_one_nccl_id():
    """The torch.distributed plumbing bench.py uses for N > 1: every rank
    gets world / rank / device from the process group and the SAME
    128-byte NCCL unique id (generated on rank 0, broadcast)."""
    import __graft_entry__
    __graft_entry__._product_build()
    ctx = mp.get_context("spawn")
    errq, outq = ctx.SimpleQueue(), ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_opts_worker, args=(r, 2, port, errq, outq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    got = sorted(outq.get() for _ in range(2))
    assert [g[:6] for g in got] == [(0, 2, 0, 0, 1, 2), (1, 2, 1, 1, 1, 2)]
    assert got[0][6] == got[1][6] and any(got[0][6])
