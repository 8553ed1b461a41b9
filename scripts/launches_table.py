"""Print an ncu --csv launch list (gpu__time_duration + optional DRAM/issue metrics) as a table."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.OrderedDict()
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    if not d["ID"].isdigit():
        continue
    e = data.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d["Grid Size"]})
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = 0.0
for k, v in data.items():
    t = v.get("gpu__time_duration.sum", 0) / 1e6
    tot += t
    b = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
    name = v["name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    extra = " ".join(f"{m.split('.')[0].split('__')[-1][:10]}={v[m]:.1f}" for m in v
                     if m.endswith("pct") or m.endswith("pct_of_peak_sustained_active"))
    print(f"{k:3d} {t:8.3f} ms {b / 1e9:8.2f} GB {b / 1e9 / max(t, 1e-9):6.2f} TB/s {v['grid']:>14s} {name[:60]:60s} {extra}")
print(f"total {tot:.3f} ms")
