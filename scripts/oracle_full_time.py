"""Wall time of the oracle (fold-children DP, OpenMP on this host's cores) for
ONE colouring of each BASELINE.json config at FULL size where the host's RAM
allows (configs 0-3; configs[4]'s tables need ~0.3-0.65 TB).  For
BASELINE.md section 4; not a bench line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

for ci in (0, 1, 2, 3):
    cfg = synth.CONFIGS[ci]
    g = cfg.graph()
    col = oracle.color(g.n, cfg.k, cfg.color_seed)
    num = oracle.NUM_EXACT if ci == 0 else (oracle.NUM_LONGDOUBLE if ci == 1 else oracle.NUM_DOUBLE)
    t = time.perf_counter()
    x = oracle.dp_count(g, cfg.parent, col, num).total
    dt = time.perf_counter() - t
    print(json.dumps({"config": ci, "name": cfg.name, "oracle_s": round(dt, 3), "cores": os.cpu_count(),
                      "colorful_maps": float(x), "numtype": num}), flush=True)
