"""Summarise an ncu --metrics gpu__time_duration.sum CSV: the last step's launches."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_last = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        h = r
        start = i + 1
        break
idx, mv, un = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
ks = [(r[idx], float(r[mv].replace(",", "")), r[un]) for r in rows[start:] if len(r) > mv]
tot = 0.0
for k, v, u in ks[-n_last:]:
    ms = v / 1e6 if u == "ns" else v / 1e3 if u == "us" else v
    tot += ms
    print(f"{ms:10.3f}  {k[:90]}")
print(f"{tot:10.3f}  total of the last {n_last}")
