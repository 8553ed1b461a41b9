"""Sampled-output vertices of the configs[4] graph for the full-size parity
checks of tests/test_gpu_config4.py (the same selection as its
_root_samples): the oracle's root count X_v (or_dp_root_at, whose work is
about sum of degrees over the radius-2 ball x 15 columns) for the configs[4]
template and the k = 16 template, with its time.  Host-only."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from test_gpu_config4 import PAR16, _root_samples  # noqa: E402

t = time.time()
g = synth.CONFIGS[4].graph()
print("gen", round(time.time() - t, 1), flush=True)
t = time.time()
samples = _root_samples(g, 6)
print("samples", samples, "s", round(time.time() - t, 1), flush=True)
for v in samples:
    for name, par, k in (("c4", synth.CONFIGS[4].parent, 15), ("k16", PAR16, 16)):
        t = time.time()
        x = oracle.dp_root_at(g, par, oracle.color(g.n, k, 2), int(v), oracle.NUM_DOUBLE)
        print(v, name, "Xv", x, "s", round(time.time() - t, 1), flush=True)
