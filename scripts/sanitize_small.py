"""compute-sanitizer target (one tool per run): configs[0] and configs[1]
(fp64 and fp32), heavy segments forced (segment_len 64), the memory plan's
batched tail with recomputation forced, column chunks, and a 2-rank loopback
partition -- every kernel family of the hot path, on small inputs.  Prints
the counts; the sanitizer's own summary decides."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1804_09764_b200 as cc  # noqa: E402
import synth  # noqa: E402
from gpu_util import context  # noqa: E402

for ci in (0, 1):
    cfg = synth.CONFIGS[ci]
    g = cfg.graph()
    for prec in ("fp64", "fp32"):
        for kw, knobs in (({}, {}), ({"segment_len": 64}, {}), ({"chunk_cols": 8}, {}),
                          ({}, {"tail_batches": 3, "tail_recompute_cols": 8}), ({}, {"gather_impl": 1}),
                          ({}, {"gather_impl": 2, "combine_impl": 2})):
            with context(g, cfg.parent, prec, **kw) as ctx:
                for name, v in knobs.items():
                    cc.cc_set_knob(ctx, name, v)
                cc.cc_color(ctx, cfg.color_seed)
                print(ci, prec, kw, knobs, cc.cc_count_colorful(ctx), flush=True)
# 2-rank loopback partition (pack kernel, remote passes), grouped and chunked
from test_gpu_loopback import run_ranks  # noqa: E402
cfg = synth.CONFIGS[1]
g = cfg.graph()
for kw in ({"exchange": 1}, {"exchange": 2, "chunk_cols": 8}):
    out, _ = run_ranks(g, cfg.parent, 2, seed=cfg.color_seed, **kw)
    print("loopback", kw, out, flush=True)
