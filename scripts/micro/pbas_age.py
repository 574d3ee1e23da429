"""PBAS per-frame cost vs. model age: T adapts (pbas.py:456-465) and with it
the update probability 1/T, so the self/neighbour-update work per frame
grows over hundreds of frames on a static background.  8 x 1080p streams,
regime T, frames timed in windows of 50 with CUDA events."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200.config import PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine, torch_stream_handle  # noqa: E402

w, h, S = 1920, 1080, 8
dev = torch.device("cuda", 0)
eng = MultiStreamEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20)), w, h, S,
                        device=0, seeds=[i + 1 for i in range(S)])
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # K2 variant: 0 auto, 1 rows, 2 strips
if mode:
    from paper_2002_00250_b200 import _native  # noqa: E402
    for e in eng.engines:
        _native.check(_native.lib().rgbdseg_pbas_set_k2_mode(e._h.ptr, mode))
ring = torch.from_numpy(_gen_ring("T", w, h, list(range(S)), 8)).to(dev)
masks = torch.empty((S, h, w), dtype=torch.uint8, device=dev)
R = ring.shape[1]
npix = w * h
st = torch_stream_handle(dev)
out = []
t = 0
marks = [40, 100, 150, 200, 300, 400, 600, 1000]
for m in marks:
    while t < m:
        eng.step_ptrs([ring.data_ptr() + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                      [masks.data_ptr() + i * npix for i in range(S)], st)
        t += 1
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        eng.step_ptrs([ring.data_ptr() + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                      [masks.data_ptr() + i * npix for i in range(S)], st)
        t += 1
    b.record()
    torch.cuda.synchronize()
    T = eng.engines[0].state_arrays()["t"]
    out.append({"mode": mode, "frame": m, "ms_per_frame": a.elapsed_time(b) / 50,
                "T_median": float(np.median(T)), "T_p10": float(np.percentile(T, 10))})
    print(json.dumps(out[-1]), flush=True)
