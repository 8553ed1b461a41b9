"""Sampled-output vertices of the configs[4] graph for the full-size parity
checks: vertices whose ball of radius 3 is small enough for the oracle's
or_dp_root_at (root counts of depth-3 templates depend only on that ball).
Host-only (the generator and numpy); prints (degree-sum bound, vertex, 2-ball
size, 3-ball size) and the oracle's X_v for the configs[4] template and the
k = 16 template of tests/test_gpu_config4.py."""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from test_gpu_config4 import PAR16, ball, induced  # noqa: E402

t = time.time()
g = synth.CONFIGS[4].graph()
print("gen", round(time.time() - t, 1), flush=True)
deg = g.degrees()
rng = np.random.default_rng(7)
cand = np.flatnonzero((deg >= 3) & (deg <= 6))
rng.shuffle(cand)
found = []
for v in cand[:400000]:
    nb = g.neighbors(int(v))
    if 1 + nb.size + int(deg[nb].sum()) > 6000:
        continue
    b2 = ball(g, int(v), 2)
    s3 = int(deg[b2].sum())
    if s3 <= 400000:
        found.append((s3, int(v), int(b2.size)))
found.sort()
print(found[:12], flush=True)
for s3, v, _ in found[:6]:
    b3 = ball(g, v, 3)
    sub = induced(g, b3)
    pos = int(np.searchsorted(b3, v))
    t = time.time()
    for name, par, k in (("c4", synth.CONFIGS[4].parent, 15), ("k16", PAR16, 16)):
        x = oracle.dp_root_at(sub, par, oracle.color(g.n, k, 2)[b3], pos, oracle.NUM_DOUBLE)
        print(v, name, "b3", b3.size, "m", sub.nnz, "Xv", x, "s", round(time.time() - t, 1), flush=True)
