"""Metric table of every kernel in an ncu report (for profiles/).

usage: python tools/ncu_summary.py REPORT.ncu-rep [title]
"""
import csv, io, subprocess, sys

M = [  # (metric, label); values printed in the report's own units (second header row)
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%pk"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor%"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_inst%"),
    ("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "fp64pipe%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("lts__t_sector_hit_rate.pct", "L2hit%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
print(f"# {sys.argv[2] if len(sys.argv) > 2 else rep}")
print("# source: ncu --set full --clock-control none (cold-cache replay; per-launch times are serialised)")
units = rows[1]
print("kernel | " + " | ".join(f"{lab}[{units[idx[m]]}]" if m in idx and units[idx[m]] else lab for m, lab in M))
for r in rows[2:]:
    name = r[idx["Kernel Name"]][:70]
    vals = []
    for m, lab in M:
        i = idx.get(m)
        if i is None or not r[i]:
            vals.append("-")
            continue
        try:
            vals.append(f"{float(r[i].replace(',', '')):.4g}")
        except ValueError:
            vals.append(r[i])
    print(name + " | " + " | ".join(vals))
