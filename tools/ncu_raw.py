"""Pipe / shared-memory / stall metrics of the kernels in an ncu report (raw page), one block per kernel.

usage: python tools/ncu_raw.py REPORT.ncu-rep
"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
keys = ("pipe", "bank_conflict", "data_bank", "issue_active", "issue_stalled", "wavefronts_mem_shared", "lsu", "mio",
        "throughput.avg.pct", "inst_executed.sum", "achieved_occupancy", "warps_active", "xbar", "lts__t_sectors_op",
        "l1tex__m_", "dram__throughput", "lts__throughput", "l1tex__throughput", "sm__throughput")
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:100])
    for i, name in enumerate(h):
        n = name.lower()
        if any(k in n for k in keys):
            try:
                val = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if val != 0:
                print(f"  {name:108s} {u[i]:14s} {r[i]}")
