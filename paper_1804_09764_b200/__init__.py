"""B200-native colour-coding tree-template counting (arXiv 1804.09764 hot path).

Thin Python binding of the C ABI in include/cc.h (libcc.so): the functions
below have the C names and only marshal arguments (numpy arrays -> host
pointers).  All computation runs in the library's sm_100a kernels; there is no
CPU fallback -- if libcc.so is missing this package fails to import.

PyTorch is used only as plumbing: `distributed_options()` broadcasts the NCCL
unique id over an existing torch.distributed process group.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from ._native import (CC_ERR_ARG, CC_ERR_CUDA, CC_ERR_GRAPH, CC_ERR_NCCL, CC_ERR_NONFINITE,  # noqa: F401
                      CC_ERR_OOM, CC_ERR_STATE, CC_ERR_TEMPLATE, CC_EXCHANGE_AUTO, CC_EXCHANGE_GROUPED,
                      CC_EXCHANGE_RING, CC_EXCHANGE_ALLTOALL, CC_EXCHANGE_DEVICE, CC_FP32, CC_FP64, CC_OK, STATUS_NAMES,
                      cc_options)

_lib = _native.lib
LIB_PATH = _native.LIB_PATH

# Phases reported by cc_last_profile (ms), in order.
PROFILE_FIELDS = ["total", "color", "csort", "hist", "gather", "combine", "root", "exchange", "exposed_exchange"]


class CCError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


def _check(ctx, st):
    if st != CC_OK:
        msg = _lib.cc_last_error(ctx).decode() if ctx else ""
        raise CCError(st, msg)


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


# ------------------------------------------------------------------ options / lifetime
def cc_default_options(**kw) -> cc_options:
    o = cc_options()
    _check(None, _lib.cc_default_options(ctypes.byref(o)))
    for k, v in kw.items():
        if k == "precision" and isinstance(v, str):
            v = {"fp64": CC_FP64, "fp32": CC_FP32}[v]
        setattr(o, k, v)
    return o


def cc_nccl_selftest(device: int = 0) -> None:
    """Test hook: one-rank NCCL grouped send/recv + all-reduce on `device`."""
    _check(None, _lib.cc_nccl_selftest(device))


def cc_nccl_device_selftest(device: int = 0) -> None:
    """Test hook: NCCL device API (symmetric window, LSA pointer, LSA barrier) on one rank."""
    _check(None, _lib.cc_nccl_device_selftest(device))


def cc_loopback_create(world: int) -> ctypes.c_void_p:
    """Test hook: an in-process transport group for `world` rank threads (cc_options.loopback)."""
    h = ctypes.c_void_p()
    _check(None, _lib.cc_loopback_create(world, ctypes.byref(h)))
    return h


def cc_loopback_destroy(group) -> None:
    _lib.cc_loopback_destroy(group)


def cc_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(None, _lib.cc_nccl_unique_id(buf))
    return buf.raw


def cc_create(opt: cc_options | None = None, **kw) -> ctypes.c_void_p:
    if opt is None:
        opt = cc_default_options(**kw)
    h = ctypes.c_void_p()
    st = _lib.cc_create(ctypes.byref(opt), ctypes.byref(h))
    if st != CC_OK:
        raise CCError(st, "cc_create failed")
    return h


def cc_destroy(ctx) -> None:
    _lib.cc_destroy(ctx)


def cc_last_error(ctx) -> str:
    return _lib.cc_last_error(ctx).decode()


# ------------------------------------------------------------------ the five calls
def cc_load_graph(ctx, n: int, row_ptr, col) -> None:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    _check(ctx, _lib.cc_load_graph(ctx, int(n), _p(rp), _p(cl)))


def cc_set_template(ctx, parent) -> None:
    par = np.ascontiguousarray(parent, dtype=np.int32)
    _check(ctx, _lib.cc_set_template(ctx, len(par), _p(par)))


def cc_set_template_colors(ctx, parent, colours: int) -> None:
    par = np.ascontiguousarray(parent, dtype=np.int32)
    _check(ctx, _lib.cc_set_template_colors(ctx, int(par.size), _p(par), int(colours)))


def cc_color(ctx, seed: int) -> None:
    _check(ctx, _lib.cc_color(ctx, seed & 0xFFFFFFFFFFFFFFFF))


def cc_count_colorful(ctx) -> float:
    x = ctypes.c_double()
    _check(ctx, _lib.cc_count_colorful(ctx, ctypes.byref(x)))
    return x.value


def cc_count_colorful_multi(ctx, parents) -> np.ndarray:
    """Colourful maps of each template (list of parent arrays) for the current colouring."""
    sizes = np.array([len(p) for p in parents], dtype=np.int32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.int32) for p in parents]), dtype=np.int32)
    out = np.zeros(len(parents), dtype=np.float64)
    _check(ctx, _lib.cc_count_colorful_multi(ctx, int(sizes.size), _p(sizes), _p(flat), _p(out)))
    return out


def cc_estimate(ctx, iterations: int, seed0: int, per_iter: bool = False):
    est = ctypes.c_double()
    xs = np.zeros(iterations, dtype=np.float64)
    _check(ctx, _lib.cc_estimate(ctx, iterations, seed0 & 0xFFFFFFFFFFFFFFFF, ctypes.byref(est), _p(xs)))
    return (est.value, xs) if per_iter else est.value


# ------------------------------------------------------------------ hooks
def cc_set_colors(ctx, colors) -> None:
    c = np.ascontiguousarray(colors, dtype=np.uint8)
    _check(ctx, _lib.cc_set_colors(ctx, _p(c)))


def cc_get_colors(ctx, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint8)
    _check(ctx, _lib.cc_get_colors(ctx, _p(out)))
    return out


def cc_template_info(ctx):
    aut, aut_root, ns = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    _check(ctx, _lib.cc_template_info(ctx, ctypes.byref(aut), ctypes.byref(aut_root), ctypes.byref(ns)))
    return aut.value, aut_root.value, ns.value


def cc_get_subtree_counts(ctx, x: int, n: int, k: int, size: int) -> np.ndarray:
    out = np.zeros((n, math.comb(k, size)), dtype=np.float64)
    _check(ctx, _lib.cc_get_subtree_counts(ctx, x, _p(out)))
    return out


def cc_set_knob(ctx, name: str, value: int) -> None:
    """Implementation knob of this context (every value computes the same result)."""
    _check(ctx, _lib.cc_set_knob(ctx, name.encode(), int(value)))


def cc_get_knob(ctx, name: str) -> int:
    v = ctypes.c_int32()
    _check(ctx, _lib.cc_get_knob(ctx, name.encode(), ctypes.byref(v)))
    return v.value


def cc_set_profiling(ctx, on: bool) -> None:
    _check(ctx, _lib.cc_set_profiling(ctx, 1 if on else 0))


def cc_last_profile(ctx) -> dict:
    buf = np.zeros(16, dtype=np.float64)
    n = ctypes.c_int32()
    _check(ctx, _lib.cc_last_profile(ctx, _p(buf), 16, ctypes.byref(n)))
    return dict(zip(PROFILE_FIELDS, buf[:n.value].tolist()))


def cc_estimate_mom(ctx, iterations: int, seed0: int, groups: int, per_iter: bool = False):
    est = ctypes.c_double()
    xs = np.zeros(iterations, dtype=np.float64)
    _check(ctx, _lib.cc_estimate_mom(ctx, iterations, seed0, groups, ctypes.byref(est), _p(xs)))
    return (est.value, xs) if per_iter else est.value


def cc_median_of_means(xs, k: int, aut: int, groups: int) -> float:
    x = np.ascontiguousarray(xs, dtype=np.float64)
    out = ctypes.c_double()
    _check(None, _lib.cc_median_of_means(_p(x), int(x.size), k, aut, groups, ctypes.byref(out)))
    return out.value


def cc_niter(eps: float, delta: float, k: int, constant: float = 1.0) -> int:
    out = ctypes.c_int64()
    _check(None, _lib.cc_niter(eps, delta, k, constant, ctypes.byref(out)))
    return out.value


def cc_get_subtree_rows(ctx, x: int, vertices, k: int, s: int) -> np.ndarray:
    """Rows of the full-subtree table of template vertex x for the given original vertex ids."""
    vs = np.ascontiguousarray(vertices, dtype=np.int32)
    w = math.comb(k, s)
    out = np.zeros((vs.size, w), dtype=np.float64)
    _check(ctx, _lib.cc_get_subtree_rows(ctx, int(x), _p(vs), int(vs.size), _p(out)))
    return out


def cc_last_stats(ctx) -> dict:
    buf = np.zeros(16, dtype=np.float64)
    _check(ctx, _lib.cc_last_stats(ctx, _p(buf), 16))
    return dict(updates=buf[0], model_bytes=buf[1], agg_bytes=buf[2], launches=buf[3], peak_table_bytes=buf[4],
                fused_root=int(buf[5]), top_gather_bytes=buf[6], top_gather_ms=buf[7], gather_launches=int(buf[8]),
                halo_bytes=buf[9], exchange=int(buf[10]), column_chunks=int(buf[11]), tail_batches=int(buf[12]),
                recompute_cols=int(buf[13]), top_gather_ordinal=int(buf[14]), sibling_pairs=int(buf[15]))


# ------------------------------------------------------------------ host-only
def cc_colex_rank(mask: int) -> int:
    return _lib.cc_colex_rank(mask)


def cc_colex_unrank(s: int, r: int) -> int:
    return _lib.cc_colex_unrank(s, r)


def cc_split_table(k: int, t: int, a: int) -> np.ndarray:
    out = np.zeros(math.comb(k, t) * math.comb(t, a), dtype=np.uint32)
    _check(None, _lib.cc_split_table(k, t, a, _p(out), out.size))
    return out.reshape(math.comb(t, a), math.comb(k, t))


def cc_zblock_table(K: int, ts: int, as_: int) -> np.ndarray:
    nb, ld = ctypes.c_int32(), ctypes.c_int32()
    _check(None, _lib.cc_zblock_table(K, ts, as_, None, 0, ctypes.byref(nb), ctypes.byref(ld)))
    out = np.zeros(nb.value * ld.value, dtype=np.uint16)
    _check(None, _lib.cc_zblock_table(K, ts, as_, _p(out), out.size, ctypes.byref(nb), ctypes.byref(ld)))
    return out.reshape(nb.value, ld.value)


def cc_plan_template(parent) -> dict:
    par = np.ascontiguousarray(parent, dtype=np.int32)
    steps = np.zeros((64, 6), dtype=np.int32)
    ns, aut, aut_root = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    mem, comp = ctypes.c_double(), ctypes.c_double()
    _check(None, _lib.cc_plan_template(len(par), _p(par), _p(steps), 64, ctypes.byref(ns), ctypes.byref(aut),
                                       ctypes.byref(aut_root), ctypes.byref(mem), ctypes.byref(comp)))
    st = [dict(zip(("t", "a", "p", "active", "passive", "out"), map(int, r))) for r in steps[:ns.value]]
    return dict(steps=st, aut=aut.value, aut_root=aut_root.value, memory=mem.value, computation=comp.value)


def cc_plan_template_auto(parent, avg_degree: float = 32.0, elem: int = 4) -> dict:
    par = np.ascontiguousarray(parent, dtype=np.int32)
    steps = np.zeros((64, 6), dtype=np.int32)
    ns, root, cost = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    _check(None, _lib.cc_plan_template_auto(len(par), _p(par), avg_degree, elem, _p(steps), 64, ctypes.byref(ns),
                                            ctypes.byref(root), ctypes.byref(cost)))
    st = [dict(zip(("t", "a", "p", "active", "passive", "out"), map(int, r))) for r in steps[:ns.value]]
    return dict(steps=st, root=root.value, cost=cost.value)


def cc_partition_plan(n: int, row_ptr, col, world: int, rank: int, relabel_seed: int = 0x5eed) -> dict:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    sizes = np.zeros(4, dtype=np.int64)
    args = (n, _p(rp), _p(cl), world, rank, relabel_seed)
    _check(None, _lib.cc_partition_plan(*args, _p(sizes), None, None, None, None, None, None, None))
    n_own, n_halo, nnz, nsend = map(int, sizes)
    own = np.zeros(n_own, np.int32)
    halo = np.zeros(n_halo, np.int32)
    recv_off = np.zeros(world + 1, np.int64)
    send_off = np.zeros(world + 1, np.int64)
    send_idx = np.zeros(nsend, np.int32)
    lrp = np.zeros(n_own + 1, np.int64)
    lcol = np.zeros(nnz, np.int32)
    _check(None, _lib.cc_partition_plan(*args, _p(sizes), _p(own), _p(halo), _p(recv_off), _p(send_off),
                                        _p(send_idx), _p(lrp), _p(lcol)))
    return dict(own_orig=own, halo_orig=halo, recv_off=recv_off, send_off=send_off, send_idx=send_idx,
                rp=lrp, col=lcol)


def cc_exchange_model(n: int, row_ptr, col, world: int, rank: int, row_bytes: float = 1024.0,
                      relabel_seed: int = 0x5eed) -> dict:
    """The cost model behind CC_EXCHANGE_AUTO for one rank (host only)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    out = np.zeros(4, dtype=np.float64)
    _check(None, _lib.cc_exchange_model(n, _p(rp), _p(cl), world, rank, relabel_seed, float(row_bytes), _p(out)))
    return dict(grouped_s=out[0], ring_s=out[1], link_bps=out[2], gather_bps=out[3])


# ------------------------------------------------------------------ torch.distributed plumbing
def distributed_options(**kw) -> tuple[cc_options, ctypes.Array]:
    """Options for this rank of an initialised torch.distributed job: world,
    rank, device = LOCAL_RANK, and the NCCL unique id broadcast from rank 0.
    Returns (options, id buffer); keep the buffer alive until cc_create."""
    import os

    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    obj = [cc_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    buf = ctypes.create_string_buffer(obj[0], 128)
    opt = cc_default_options(world=world, rank=rank, device=int(os.environ.get("LOCAL_RANK", rank)), **kw)
    opt.nccl_id = ctypes.cast(buf, ctypes.c_void_p)
    return opt, buf
