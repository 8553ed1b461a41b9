"""Measurement of cc_count_colorful_multi: all unlabelled trees on
k vertices on one colouring, with the cross-template table cache, against one
cc_count_colorful per template.  GPU.  Prints one JSON line."""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_09764_b200 as cc  # noqa: E402
import synth  # noqa: E402


def unrooted_code(parent):
    k = len(parent)
    adj = [[] for _ in range(k)]
    for v, p in enumerate(parent):
        if p >= 0:
            adj[v].append(p)
            adj[p].append(v)

    def code(x, frm):
        return "(" + "".join(sorted(code(y, x) for y in adj[x] if y != frm)) + ")"
    return min(code(r, -1) for r in range(k))


def all_trees(k):
    seen, out = set(), []
    for tail in itertools.product(*[range(i) for i in range(1, k)]):
        par = [-1] + list(tail)
        c = unrooted_code(par)
        if c not in seen:
            seen.add(c)
            out.append(par)
    return out


ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--k", type=int, default=7)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
cfg = synth.CONFIGS[args.config]
g = cfg.graph()
trees = all_trees(args.k)
ctx = cc.cc_create(device=0, precision=cc.CC_FP32)
cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
cc.cc_set_template(ctx, trees[0])
cc.cc_color(ctx, 2)
cc.cc_count_colorful_multi(ctx, trees)  # warm
t_multi = []
for _ in range(args.reps):
    t = time.perf_counter()
    xs = cc.cc_count_colorful_multi(ctx, trees)
    t_multi.append(time.perf_counter() - t)
reused = cc.cc_last_stats(ctx)["halo_bytes"]
t_single = []
for _ in range(args.reps):
    t = time.perf_counter()
    ys = []
    for par in trees:
        cc.cc_set_template(ctx, par)
        cc.cc_color(ctx, 2)
        ys.append(cc.cc_count_colorful(ctx))
    t_single.append(time.perf_counter() - t)
cc.cc_destroy(ctx)
same = all(abs(a - b) <= 1e-4 * abs(b) for a, b in zip(xs, ys))
print(json.dumps({"workload": f"configs[{args.config}] graph, all {len(trees)} trees on {args.k} vertices, fp32",
                  "multi_ms": 1e3 * min(t_multi), "single_templates_ms": 1e3 * min(t_single),
                  "speedup": min(t_single) / min(t_multi), "tables_reused": reused, "counts_agree": same}))
