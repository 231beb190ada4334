"""Summarise the hottest SASS lines (by stall samples) of one kernel in an ncu report.

usage: python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
print(lines[0])
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[1:]:
    try:
        n = int(r[si])
    except ValueError:
        continue
    tops = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i]) for i in stall_cols), reverse=True)[:2]
    data.append((n, r[0][-5:], r[1].strip()[:70], tops))
tot = sum(d[0] for d in data)
print("total samples", tot)
for n, a, s, t in sorted(data, reverse=True)[:top]:
    print(f"{n:7d} {100*n/tot:5.1f}% {a} {s:70s} {t}")
