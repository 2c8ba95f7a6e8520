"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel.

    python tools/launch_summary.py launches.csv > summary.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
agg = OrderedDict()
for r in rows:
    name = r[4].split("(")[0] if "(" in r[4] else r[4]
    us = float(r[14]) / (1000.0 if r[13] == "ns" else 1.0)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + us)
total = sum(t for _, t in agg.values())
print("kernel,launches,total_us,share")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k},{n},{t:.1f},{t / total:.4f}")
