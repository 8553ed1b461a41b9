"""Tuning sweep (GPU): per-phase device ms of one colouring for each
aggregation-kernel variant / chunk width / segment length.  Not a bench."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_09764_b200 as cc  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--variants", default="0,1,2,4")
ap.add_argument("--segs", default="4096")
ap.add_argument("--chunks", default="0")
ap.add_argument("--precision", default=None)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()

cfg = synth.CONFIGS[args.config]
t = time.time()
g = cfg.graph()
print(f"graph {cfg.name}: n={g.n} 2m={g.nnz} gen {time.time() - t:.1f}s", flush=True)
prec = args.precision or cfg.precision
for seg in map(int, args.segs.split(",")):
    for chunk in map(int, args.chunks.split(",")):
        ctx = cc.cc_create(device=0, precision=cc.CC_FP32 if prec == "fp32" else cc.CC_FP64, segment_len=seg,
                           chunk_cols=chunk)
        t = time.time()
        cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
        cc.cc_set_template(ctx, cfg.parent)
        load_s = time.time() - t
        for var in args.variants.split(","):
            os.environ["CC_GATHER_VARIANT"] = var
            cc.cc_color(ctx, 2)
            cc.cc_count_colorful(ctx)  # warm
            best = None
            for r in range(args.reps):
                cc.cc_color(ctx, 2 + r)
                x = cc.cc_count_colorful(ctx)
                p = cc.cc_last_profile(ctx)
                if best is None or p["total"] < best["total"]:
                    best = p
            st = cc.cc_last_stats(ctx)
            print(json.dumps({"variant": var, "seg": seg, "chunk": chunk, "load_s": round(load_s, 1),
                              "agg_GBs": round(st["agg_bytes"] / best["gather"] / 1e6, 1),
                              **{k: round(v, 3) for k, v in best.items()}}), flush=True)
        cc.cc_destroy(ctx)
