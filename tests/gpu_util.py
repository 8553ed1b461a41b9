"""Helpers for the -m gpu parity tests: drive the CUDA path through the C ABI."""
from __future__ import annotations

import contextlib
import math

import numpy as np


def lib():
    import paper_1804_09764_b200 as cc
    return cc


@contextlib.contextmanager
def context(g, parent, precision="fp64", **opts):
    cc = lib()
    ctx = cc.cc_create(device=0, precision=cc.CC_FP64 if precision == "fp64" else cc.CC_FP32, **opts)
    try:
        cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
        cc.cc_set_template(ctx, parent)
        yield ctx
    finally:
        cc.cc_destroy(ctx)


def count(g, parent, colors=None, seed=None, precision="fp64", **opts) -> float:
    cc = lib()
    with context(g, parent, precision, **opts) as ctx:
        if colors is not None:
            cc.cc_set_colors(ctx, colors)
        else:
            cc.cc_color(ctx, seed)
        return cc.cc_count_colorful(ctx)


def subtree_sizes(parent):
    k = len(parent)
    size = [1] * k
    for v in range(k):
        p = parent[v]
        while p >= 0:
            size[p] += 1
            p = parent[p]
    return size


def tables(g, parent, colors, precision="fp64", **opts):
    """Every full-subtree table D_x (n x C(k, s_x), colex) from the GPU."""
    cc = lib()
    k = len(parent)
    sizes = subtree_sizes(parent)
    out = {}
    with context(g, parent, precision, **opts) as ctx:
        cc.cc_set_colors(ctx, colors)
        for x in range(k):
            if parent[x] == -1:
                out[x] = cc.cc_get_subtree_counts(ctx, x, g.n, k, k)
            else:
                out[x] = cc.cc_get_subtree_counts(ctx, x, g.n, k, sizes[x])
    return out


def assert_close_entries(got, want, rel, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    zero = want == 0
    assert np.all(got[zero] == 0), f"{what}: nonzero where the oracle has 0"
    nz = ~zero
    if nz.any():
        err = np.abs(got[nz] - want[nz]) / np.abs(want[nz])
        assert err.max() <= rel, f"{what}: max rel err {err.max():.3e} > {rel:.1e}"


def rel_err(a, b) -> float:
    return abs(a - b) / abs(b) if b else abs(a)


def comb(k, s):
    return math.comb(k, s)
