#!/usr/bin/env python
"""Per-opcode and per-region dynamic instruction counts of one kernel from an
ncu report (source page, SASS view).  usage: sass_hist.py REP [--dump FILE]"""
import csv, collections, io, re, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, src, th = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Avg. Threads Executed")
data = [(int(r[ie] or 0), r[th], r[src].strip()) for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
warps = data[0][0]
tot = sum(n for n, _, _ in data)
print(f"warps {warps}  instr/warp {tot / warps:.1f}")
by = collections.Counter()
for n, _, s in data:
    by[re.sub(r'^@!?U?P\w+\s+', '', s).split(' ')[0].split('.')[0]] += n
for op, n in by.most_common(30):
    print(f"  {op:12s} {n / warps:7.1f}")
if "--dump" in sys.argv:
    with open(sys.argv[sys.argv.index("--dump") + 1], "w") as f:
        for i, (n, t, s) in enumerate(data):
            f.write(f"{i} {n / warps:.3f} {t} {s}\n")
