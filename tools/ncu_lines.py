"""Hottest CUDA source lines (warp stall samples and executed warp instructions) of one kernel in
an ncu report captured with --import-source on (kernels built with -lineinfo).

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]
"""
import csv, io, os, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data, fname, hdr = [], "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
    elif r[0] == "Function Name":
        func = r[1]
    elif r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    elif hdr and r[0].isdigit():
        n = int(r[si]) if r[si].isdigit() else 0
        ins = int(r[ii]) if r[ii].isdigit() else 0
        tops = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
        data.append((n, ins, fname, r[0], r[1].strip()[:84], tops))
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"# {func[:120]}")
print(f"# total stall samples {tot}, warp instructions executed {toti}")
for n, ins, f, ln, s, t in sorted(data, reverse=True)[:top]:
    print(f"{100*n/tot:5.1f}% inst {100*ins/toti:5.1f}% {f}:{ln:<5} {s:84s} {t}")
