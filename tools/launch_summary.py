"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (dev tool):
python tools/launch_summary.py launches.csv "header line" > summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.OrderedDict()
for r in rows[1:]:
    us = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(r[ui], 1e-3)
    n, t = tot.get(r[ki], (0, 0.0))
    tot[r[ki]] = (n + 1, t + us)
s = sum(t for _, t in tot.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print(f"{'kernel':110s} launches   total_us  share")
for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:110]:110s} {n:8d} {t:10.1f} {100 * t / s:5.1f}%")
