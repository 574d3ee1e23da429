"""8 x 1080p PBAS burned in for --frames frames (T reaches t_lower = 2 after
~300), then 5 more frames: run under ncu to split the long-run frame cost."""
import sys

import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200.config import PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine, torch_stream_handle  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 450
w, h, S = 1920, 1080, 8
dev = torch.device("cuda", 0)
eng = MultiStreamEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20)), w, h, S,
                        device=0, seeds=[i + 1 for i in range(S)])
ring = torch.from_numpy(_gen_ring("T", w, h, list(range(S)), 8)).to(dev)
masks = torch.empty((S, h, w), dtype=torch.uint8, device=dev)
R, npix, st = ring.shape[1], w * h, torch_stream_handle(dev)
if "tiles" in sys.argv[2:]:  # pin the tile K2 (profilers replay kernels; auto mode reads host memory)
    from paper_2002_00250_b200 import _native

    for e in eng.engines:
        _native.check(_native.lib().rgbdseg_pbas_set_k2_mode(e._h.ptr, 2))
for t in range(frames + 5):
    eng.step_ptrs([ring.data_ptr() + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                  [masks.data_ptr() + i * npix for i in range(S)], st)
torch.cuda.synchronize()
