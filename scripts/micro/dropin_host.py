"""Drop-in host path: SegmentationEngine.process_frame(numpy) on one 1920x1080
RGB-D stream through GMM 7/3 and PBAS n=20 (the call process_sequence and the
reference's service make per frame; engine.py:99-112).  Host frames in,
host masks out.  Prints ms per frame (both algorithms) and Mpixel/s."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2002_00250_b200 import synth  # noqa: E402
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import SegmentationEngine  # noqa: E402

w, h = 1920, 1080
frames = [synth.make_frame("T", w, h, 0, t) for t in range(8)]
g = SegmentationEngine(PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=7, k_d=3)), w, h)
p = SegmentationEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20), seed=1), w, h)
for t in range(45):
    g.process_frame(frames[t % 8])
    p.process_frame(frames[t % 8])
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
t0 = time.perf_counter()
for t in range(N):
    mg = g.process_frame(frames[t % 8])
    mp = p.process_frame(frames[t % 8])
dt = (time.perf_counter() - t0) / N
print(json.dumps({"ms_per_frame": dt * 1e3, "mpix_s": w * h / dt / 1e6, "frames": N}))
