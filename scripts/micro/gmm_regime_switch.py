"""GMM K1 cost when the scene changes: 8 x 1080p GMM 7/3 burned in on regime S
(every component seeded), then fed regime T frames (nothing matches at
first: every pixel takes the least-fit replacement path, gmm.py:326-337).
Prints ms per step for S frames and for the first / later T frames."""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200.config import GmmParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine, torch_stream_handle  # noqa: E402

w, h, S = 1920, 1080, 8
npix = w * h
dev = torch.device("cuda", 0)
eng = MultiStreamEngine(PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=7, k_d=3)),
                        w, h, S, device=0)
rings = {r: torch.from_numpy(_gen_ring(r, w, h, list(range(S)), 7)).to(dev) for r in ("S", "T")}
masks = torch.empty((S, h, w), dtype=torch.uint8, device=dev)
st = torch_stream_handle(dev)


def step(r, t):
    ring = rings[r]
    R = ring.shape[1]
    eng.step_ptrs([ring.data_ptr() + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                  [masks.data_ptr() + i * npix for i in range(S)], st)


def timed(r, t0, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for t in range(t0, t0 + n):
        step(r, t)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for t in range(8):
    step("S", t)
out = {"S": timed("S", 8, 20)}
out["T_first5"] = timed("T", 0, 5)
out["T_next20"] = timed("T", 5, 20)
out["T_fg_fraction"] = float((masks > 0).float().mean())
out["T_later50"] = timed("T", 25, 50)
out["T_fg_fraction_later"] = float((masks > 0).float().mean())
print(json.dumps(out))
