"""Run one configs[ci] twin count per knob setting, each in a fresh process
(a CUDA fault poisons the process): prints which settings fail.
    python scripts/knob_probe.py CI [PREC]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CHILD = r'''
import sys, os
sys.path.insert(0, %r); sys.path.insert(0, os.path.join(%r, "tests"))
import synth, oracle
import paper_1804_09764_b200 as cc
from gpu_util import context, rel_err
ci, prec, name, value = %d, %r, %r, %d
cfg = synth.scaled_twin(synth.CONFIGS[ci], 11, 16)
g = cfg.graph()
col = oracle.color(g.n, cfg.k, 23)
want = float(oracle.dp_count(g, cfg.parent, col, oracle.NUM_LONGDOUBLE).total)
with context(g, cfg.parent, prec, segment_len=64) as ctx:
    cc.cc_set_colors(ctx, col)
    if name: cc.cc_set_knob(ctx, name, value)
    x = cc.cc_count_colorful(ctx)
print("rel_err", rel_err(x, want))
'''

if __name__ == "__main__":
    from test_gpu_parity import KNOB_SETTINGS
    ci = int(sys.argv[1])
    precs = sys.argv[2:] or ["fp64", "fp32"]
    for prec in precs:
        for name, value in [("", 0)] + KNOB_SETTINGS:
            r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, ROOT, ci, prec, name, value)],
                               capture_output=True, text=True, timeout=600)
            tail = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else \
                (r.stderr.strip().splitlines() or [""])[-1][:200]
            print(f"ci={ci} {prec} {name or 'default'}={value}: rc={r.returncode} {tail}", flush=True)
