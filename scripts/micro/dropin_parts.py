"""Where the drop-in host path's time goes (1920x1080): per-call ms of
GMM / PBAS process_frame(numpy), the device step alone (CUDA tensor in/out),
and a host copy of one frame into page-locked memory."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2002_00250_b200 import synth  # noqa: E402
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import SegmentationEngine  # noqa: E402

w, h = 1920, 1080
frames = [synth.make_frame("T", w, h, 0, t) for t in range(8)]
out = {}


def per_call(fn, n=60):
    for t in range(10):
        fn(t)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(n):
        fn(t)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


for name, cfg in (("gmm", PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=7, k_d=3))),
                  ("pbas", PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20), seed=1))):
    e = SegmentationEngine(cfg, w, h)
    for t in range(45):
        e.process_frame(frames[t % 8])
    out[f"{name}_process_frame_numpy_ms"] = per_call(lambda t: e.process_frame(frames[t % 8]))
    dev = [torch.from_numpy(f).cuda() for f in frames]
    out[f"{name}_device_step_ms"] = per_call(lambda t: e.process_frame(dev[t % 8]))
    pin = [torch.from_numpy(f).pin_memory().numpy() for f in frames]
    mk = torch.empty((h, w), dtype=torch.uint8).pin_memory().numpy()

    def sub(t):
        e.submit(pin[t % 8], mk)
    out[f"{name}_submit_pinned_ms"] = per_call(lambda t: (sub(t), e.synchronize()))
    e.close()
pinbuf = torch.empty((h, w, 4), dtype=torch.uint8).pin_memory().numpy()
out["np_copy_to_pinned_ms"] = per_call(lambda t: np.copyto(pinbuf, frames[t % 8]))
out["np_copy_frame_ms"] = per_call(lambda t: frames[(t + 1) % 8].copy())
print(json.dumps(out))
