"""ms per frame of 8 x 1080p PBAS at T = t_lower (frames 450-500), K2 pinned
to the given variant (1 rows, 2 tiles)."""
import sys

import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200 import _native  # noqa: E402
from paper_2002_00250_b200.config import PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine, torch_stream_handle  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w, h, S = 1920, 1080, 8
dev = torch.device("cuda", 0)
eng = MultiStreamEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20)), w, h, S,
                        device=0, seeds=[i + 1 for i in range(S)])
for e in eng.engines:
    _native.check(_native.lib().rgbdseg_pbas_set_k2_mode(e._h.ptr, mode))
ring = torch.from_numpy(_gen_ring("T", w, h, list(range(S)), 8)).to(dev)
masks = torch.empty((S, h, w), dtype=torch.uint8, device=dev)
R, npix, st = ring.shape[1], w * h, torch_stream_handle(dev)


def step(t):
    eng.step_ptrs([ring.data_ptr() + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                  [masks.data_ptr() + i * npix for i in range(S)], st)


for t in range(450):
    step(t)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for t in range(450, 500):
    step(t)
b.record()
torch.cuda.synchronize()
print(f"mode {mode}: {a.elapsed_time(b) / 50:.4f} ms/frame at T = t_lower")
