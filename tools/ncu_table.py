"""Summarize an ncu --csv launch list (per kernel name: launches, mean us, DRAM MB per launch)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = OrderedDict()
for r in rows[1:]:
    per.setdefault(r[ii], {"name": r[ki].split("(")[0]})[r[mi]] = float(r[vi].replace(",", ""))
agg = OrderedDict()
for v in per.values():
    a = agg.setdefault(v["name"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0.0)
    a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
print(f"{'kernel':34s} {'n':>3s} {'us/launch':>10s} {'DRAM MB/launch':>15s}")
for name, (n, t, b) in agg.items():
    print(f"{name[:34]:34s} {n:3d} {t / n / 1e3:10.1f} {b / n / 1e6:15.1f}")
