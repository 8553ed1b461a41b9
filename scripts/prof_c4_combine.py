"""One count of configs[4]'s template (15-vertex binary tree, k = 15, fp32) on
an R-MAT twin, for profiling its (7;4,3) combine:
    python scripts/prof_c4_combine.py [SCALE] [EF] [REPS]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1804_09764_b200 as cc  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ef = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = synth.scaled_twin(synth.CONFIGS[4], scale, ef)
g = cfg.graph()
ctx = cc.cc_create(device=0, precision=cc.CC_FP32)
cc.cc_load_graph(ctx, g.n, g.row_ptr, g.col)
cc.cc_set_template(ctx, cfg.parent)
cc.cc_color(ctx, 2)
for i in range(reps):
    t = time.time()
    x = cc.cc_count_colorful(ctx)
    p = cc.cc_last_profile(ctx)
    print(f"count {x:.6e} wall {1e3 * (time.time() - t):.1f} ms profile {p}", flush=True)
cc.cc_destroy(ctx)
