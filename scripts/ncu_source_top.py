"""Top source lines of one kernel from `ncu -i REP --page source --csv
--print-source cuda,sass --launch-skip N --launch-count 1` output:
instructions executed and warp-stall samples per CUDA source line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
fname = ""
agg = {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        ins = float(d["Instructions Executed"])
        st = float(d["Warp Stall Sampling (All Samples)"])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    e = agg.setdefault(key, [0.0, 0.0, r[1][:90]])
    e[0] += ins
    e[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti:.3e}, stall samples {ts:.3e}")
for (f, ln), (ins, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{f}:{ln:5d} ins {100 * ins / ti:5.1f}% stall {100 * st / ts:5.1f}%  {src}")
