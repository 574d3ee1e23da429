#!/usr/bin/env python
"""Average per-kernel duration from an ncu launch list (--metrics
gpu__time_duration.sum --csv).  usage: launch_times.py launches.csv [skip]"""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d = collections.defaultdict(list)
for r in rows[1 + skip:]:
    if r[mi] == "gpu__time_duration.sum":
        d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v)/len(v):9.2f} last10={sum(v[-10:])/len(v[-10:]):9.2f}")
