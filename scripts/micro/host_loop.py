"""Host-side cost of the per-frame call on small device frames: one 640x480
stream, process_frame(CUDA tensor) in a Python loop (what a single-camera
application does), wall time per frame vs the device time per frame."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2002_00250_b200 import synth  # noqa: E402
from paper_2002_00250_b200.config import PbasParams, PipelineConfig, GmmParams  # noqa: E402
from paper_2002_00250_b200.engine import SegmentationEngine  # noqa: E402

w, h = 640, 480
frames = [torch.from_numpy(synth.make_frame("T", w, h, 0, t)).cuda() for t in range(8)]
out = {}
for algo, cfg in (("gmm", PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=3, k_d=3))),
                  ("pbas", PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20)))):
    with SegmentationEngine(cfg, w, h) as eng:
        for t in range(60):
            eng.process_frame(frames[t % 8])
        torch.cuda.synchronize()
        n = 500
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        for t in range(n):
            eng.process_frame(frames[t % 8])
        b.record()
        host = (time.perf_counter() - t0) / n
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / n
        out[algo] = {"host_us_per_call": host * 1e6, "wall_us_per_frame": wall * 1e6,
                     "gpu_us_per_frame": a.elapsed_time(b) * 1e3 / n}
print(json.dumps(out))
