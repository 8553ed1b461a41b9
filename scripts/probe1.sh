python - <<'PY'
import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import synth, oracle
import paper_1804_09764_b200 as cc
from gpu_util import context, rel_err
cfg = synth.scaled_twin(synth.CONFIGS[3], 11, 16)
g = cfg.graph()
col = oracle.color(g.n, cfg.k, 23)
for prof in [0]:
  with context(g, cfg.parent, "fp32", segment_len=64) as ctx:
    cc.cc_set_colors(ctx, col)
    cc.cc_set_knob(ctx, "gather_impl", 1)
    try:
        x = cc.cc_count_colorful(ctx)
        print("ok", x)
    except Exception as e:
        print("ERR", e)
PY
