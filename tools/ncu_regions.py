"""Stall samples of one kernel aggregated per SASS address range and reason.

usage: python tools/ncu_regions.py REPORT KERNEL_REGEX lo-hi[,lo-hi...]   (hex offsets)
"""
import csv, io, subprocess, sys
from collections import Counter, defaultdict

rep, kre, ranges = sys.argv[1], sys.argv[2], sys.argv[3]
rs = [tuple(int(x, 16) for x in r.split("-")) for r in ranges.split(",")]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
ai = hdr.index("Address")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = defaultdict(Counter)
tot = Counter()
base = None
for r in rows[1:]:
    try:
        a = int(r[ai], 16)
        n = int(r[si])
        base = a if base is None else base
        a -= base
    except ValueError:
        continue
    key = "other"
    for lo, hi in rs:
        if lo <= a < hi:
            key = f"{lo:x}-{hi:x}"
    tot[key] += n
    for i in stall_cols:
        v = int(r[i]) if r[i].isdigit() else 0
        agg[key][hdr[i]] += v
T = sum(tot.values())
for k, n in tot.most_common():
    print(f"{k:15s} {n:8d} {100*n/T:5.1f}%  ", ", ".join(f"{s[6:]}={v}" for s, v in agg[k].most_common(6)))
