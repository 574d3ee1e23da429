#!/usr/bin/env python
"""Summarise ncu captures (.ncu-rep) into a markdown table for profiles/.

usage: python scripts/ncu_summary.py OUT.md REP [REP ...]
Reads each report with `ncu -i REP --page raw --csv` and keeps the metrics
the roofline claims rest on (duration, DRAM bytes, DRAM %, occupancy, pipe
utilisation, instruction count).
"""

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    return d


def main():
    out = sys.argv[1]
    lines = ["| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " | achieved DRAM GB/s |",
             "|---|" + "---|" * (len(METRICS) + 1)]
    for rep in sys.argv[2:]:
        d = read(rep)
        name = d.get("Kernel Name", ("?", ""))[0]
        cells = []
        for key, _ in METRICS:
            v, u = d.get(key, ("n/a", ""))
            cells.append(f"{v} {u}".strip())
        try:
            def to_bytes(v, u):
                return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]

            def to_s(v, u):
                return float(v) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}[u]

            rb = to_bytes(*d["dram__bytes_read.sum"])
            wb = to_bytes(*d["dram__bytes_write.sum"])
            t = to_s(*d["gpu__time_duration.sum"])
            gbs = f"{(rb + wb) / t / 1e9:.0f}"
        except Exception:
            gbs = "n/a"
        lines.append(f"| {name[:60]} | " + " | ".join(cells) + f" | {gbs} |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
