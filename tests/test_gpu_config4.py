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


@pytest.fixture(scope="module")
def graph4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return synth.CONFIGS[4].graph()


def _ball2(g, v):
    nb = g.neighbors(v)
    verts = np.unique(np.concatenate([[v], nb] + [g.neighbors(int(u)) for u in nb]))
    return verts


def _induced(g, verts):
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
        verts = _ball2(g, v)
        sub = _induced(g, verts)
        pos = int(np.searchsorted(verts, v))
        ref = oracle.dp_count(sub, cfg.parent, col[verts], oracle.NUM_DOUBLE, keep_x=1).table[pos]
        assert ref.shape == rows[i].shape
        zero = ref == 0
        assert np.all(rows[i][zero] == 0), f"v={v}: nonzero where the oracle has 0"
        if (~zero).any():
            err = np.max(np.abs(rows[i][~zero] - ref[~zero]) / ref[~zero])
            assert err <= TOL_FP32, f"v={v}: max rel err {err:.3e}"
