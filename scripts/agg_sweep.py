"""Tuning sweep (GPU): per-phase device ms of one colouring for each kernel
variant (implementation knobs, cc_set_knob) / segment length.
Not a bench.

  --knobs "gather_impl=0,2;narrow_impl=0,4"
expands to the cartesian product of the listed values."""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_09764_b200 as cc  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--knobs", default="fused_root=1")
ap.add_argument("--segs", default="4096")
ap.add_argument("--precision", default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--check", action="store_true", help="compare every variant's count with the first")
ap.add_argument("--fixed-root", default="0")
args = ap.parse_args()

knobs = []
for part in args.knobs.split(";"):
    name, vals = part.split("=")
    knobs.append([(name, v) for v in vals.split(",")])
combos = list(itertools.product(*knobs))

cfg = synth.CONFIGS[args.config]
t = time.time()
g = cfg.graph()
print(f"graph {cfg.name}: n={g.n} 2m={g.nnz} gen {time.time() - t:.1f}s", flush=True)
prec = args.precision or cfg.precision
for seg, fr in itertools.product(map(int, args.segs.split(",")), map(int, args.fixed_root.split(","))):
    ctx = cc.cc_create(device=0, precision=cc.CC_FP32 if prec == "fp32" else cc.CC_FP64, segment_len=seg,
                       fixed_root=fr)
    t = time.time()
    cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
    cc.cc_set_template(ctx, cfg.parent)
    load_s = time.time() - t
    ref = None
    for combo in combos:
        for name, val in combo:
            cc.cc_set_knob(ctx, name, int(val))
        cc.cc_color(ctx, 2)
        cc.cc_count_colorful(ctx)  # warm
        best = None
        xs = []
        for r in range(args.reps):
            cc.cc_color(ctx, 2 + r)
            xs.append(cc.cc_count_colorful(ctx))
            p = cc.cc_last_profile(ctx)
            if best is None or p["total"] < best["total"]:
                best = p
        st = cc.cc_last_stats(ctx)
        if ref is None:
            ref = xs
        rec = {"knobs": dict(combo), "seg": seg, "fixed_root": fr, "load_s": round(load_s, 1),
               "gather_GBs": round(st["agg_bytes"] / best["gather"] / 1e6, 1),
               "same_as_first": xs == ref,
               **{k: round(v, 3) for k, v in best.items()}}
        print(json.dumps(rec), flush=True)
    cc.cc_destroy(ctx)
