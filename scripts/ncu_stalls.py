#!/usr/bin/env python
"""Issue/pipe utilisation and stall breakdown of an ncu report. usage: ncu_stalls.py REP"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = dict(zip(rows[0], rows[2]))
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    if k in d: print(f"{k:70s} {d[k]}")
st = {k.split("stalled_")[1].split("_per")[0]: float(v) for k, v in d.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
print("stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0.05))
