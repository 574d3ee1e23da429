"""Trace the auto K2 variant (1 rows / 2 tiles) and the posted update count per
frame for 8 x 1080p PBAS streams (regime T) over 500 frames."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200 import _native  # noqa: E402
from paper_2002_00250_b200.config import PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine, torch_stream_handle  # noqa: E402

w, h, S = 1920, 1080, 8
dev = torch.device("cuda", 0)
eng = MultiStreamEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20)), w, h, S,
                        device=0, seeds=[i + 1 for i in range(S)])
ring = torch.from_numpy(_gen_ring("T", w, h, list(range(S)), 8)).to(dev)
masks = torch.empty((S, h, w), dtype=torch.uint8, device=dev)
R, npix, st = ring.shape[1], w * h, torch_stream_handle(dev)
L = _native.lib()
h0 = eng.engines[0]._h.ptr
prev = None
for t in range(500):
    mode = int(L.rgbdseg_pbas_get_k2_mode(h0))
    eng.step_ptrs([ring.data_ptr() + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                  [masks.data_ptr() + i * npix for i in range(S)], st)
    if mode != prev or t % 50 == 0:
        torch.cuda.synchronize()
        print(t, mode, flush=True)
        prev = mode
