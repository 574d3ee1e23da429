#!/usr/bin/env python
"""profiles/traffic.json from ncu --set full captures of the bench's launches:
DRAM bytes (read + write) per launch, the `roofline.traffic` field of bench.py."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = {h: (v, u) for h, v, u in zip(rows[0], rows[2], rows[1])}
    r = float(d["dram__bytes_read.sum"][0]) * UNITS[d["dram__bytes_read.sum"][1]]
    w = float(d["dram__bytes_write.sum"][0]) * UNITS[d["dram__bytes_write.sum"][1]]
    return r + w


if __name__ == "__main__":
    out = Path(sys.argv[1])
    data = json.loads(out.read_text()) if out.exists() else {}
    for spec in sys.argv[2:]:  # key=report
        key, rep = spec.split("=", 1)
        data[key] = dram_bytes(rep)
    out.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data, indent=1))
