"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count / total / mean µs.

usage: python tools/launches.py LAUNCHES.csv [last_n]   (last_n: only the last n launches)
"""
import csv, sys
from collections import OrderedDict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if not l.startswith("==")]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000 if unit == "ns" else (v * 1000 if unit == "ms" else v)
        rows.append((r["Kernel Name"][:90], us))
if len(sys.argv) > 2:
    rows = rows[-int(sys.argv[2]):]
agg = OrderedDict()
for k, us in rows:
    c = agg.setdefault(k, [0, 0.0])
    c[0] += 1
    c[1] += us
tot = sum(c[1] for c in agg.values())
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us:10.1f} us {100 * us / tot:5.1f}%  n={n:4d} mean={us / n:9.1f}  {k}")
print(f"{tot:10.1f} us total over {len(rows)} launches")
