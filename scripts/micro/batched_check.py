"""Batched (one launch, 3 handles) vs single-engine GMM: mask / state mismatch
counts, for f64 and f32 state storage (diagnostic for sanitizer runs)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2002_00250_b200 import synth  # noqa: E402
from paper_2002_00250_b200.config import GmmParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine, SegmentationEngine, torch_stream_handle  # noqa: E402

w, h, n, T = 64, 48, 3, 12
for state in ("float64", "float32"):
    cfg = PipelineConfig(algorithm="gmm", gmm=GmmParams(k_rgb=7, k_d=3), gmm_state_dtype=state)
    seqs = [synth.sequence("S", w, h, seed=s, frames=T) for s in range(n)]
    ms = MultiStreamEngine(cfg, w, h, n, device=0)
    masks = torch.zeros((T, n, h, w), dtype=torch.uint8, device="cuda:0")
    frames = torch.from_numpy(np.stack([np.stack(s) for s in seqs], axis=1)).cuda()  # T, n, h, w, 4
    for t in range(T):
        ms.step_ptrs([frames[t, i].data_ptr() for i in range(n)],
                     [masks[t, i].data_ptr() for i in range(n)], torch_stream_handle())
    torch.cuda.synchronize()
    mb = masks.cpu().numpy()
    for i in range(n):
        with SegmentationEngine(cfg, w, h, device=0) as e:
            ms1 = np.stack([e.process_frame(f) for f in seqs[i]])
            st1 = {k: v.copy() for k, v in e.state_arrays().items()}
        bad = [int((mb[t, i] != ms1[t]).sum()) for t in range(T)]
        stb = ms.engines[i].state_arrays()
        sbad = {k: int((stb[k] != st1[k]).sum()) for k in st1}
        print(state, "stream", i, "mask mismatches per frame", bad, "state", sbad, flush=True)
    ms.close() if hasattr(ms, "close") else None
