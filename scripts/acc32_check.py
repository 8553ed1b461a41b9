import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle, synth
import paper_1804_09764_b200 as cc
from gpu_util import count
for ci, scale, ef in ((3, 12, 32), (3, 13, 32), (4, 11, 64)):
    cfg = synth.scaled_twin(synth.CONFIGS[ci], scale, ef)
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, 5)
    want = float(oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE).total)
    r = {}
    for a in ("0", "1"):
        os.environ["CC_ACC32"] = a
        r[a] = count(g, cfg.parent, colors=col, precision="fp32", segment_len=64)
    print(ci, scale, {a: abs(x - want) / want for a, x in r.items()})
g = synth.CONFIGS[3].graph()
col = oracle.color(g.n, 12, 2)
r = {}
for a in ("0", "1"):
    os.environ["CC_ACC32"] = a
    r[a] = count(g, synth.CONFIGS[3].parent, colors=col, precision="fp32")
print("config3 full: rel diff acc32 vs fp64 rows", abs(r["1"] - r["0"]) / r["0"])
