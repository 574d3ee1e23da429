"""Where a small single-stream PBAS step goes (K2 vs K3), cold L2 as in the
bench's config-2/3 timing: one WxH stream aged to T = t_lower, then per step
flush L2, event, classify (K2), event, apply (K3), event."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200 import _native  # noqa: E402
from paper_2002_00250_b200.config import PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle  # noqa: E402

w, h = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (640, 480)
dev = torch.device("cuda", 0)
L = _native.lib()
ring = torch.from_numpy(_gen_ring("T", w, h, [0], 8)[0]).to(dev)
mask = torch.empty((h, w), dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}
for mode, name in ((1, "rows"), (2, "strips")):
    eng = SegmentationEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20), seed=1),
                             w, h, device=0)
    _native.check(L.rgbdseg_pbas_set_k2_mode(eng._h.ptr, mode))
    st = ctypes.c_void_p(torch_stream_handle(dev))
    for t in range(400):
        eng.step_device(ring[t % 8].data_ptr(), mask.data_ptr(), st.value)
    k2, k3 = [], []
    for t in range(400, 440):
        flush.fill_(t & 255)
        flush.amax()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        fp = ctypes.c_void_p(ring[t % 8].data_ptr())
        e[0].record()
        _native.check(L.rgbdseg_pbas_classify(eng._h.ptr, fp, ctypes.c_void_p(mask.data_ptr()), st))
        e[1].record()
        _native.check(L.rgbdseg_pbas_apply(eng._h.ptr, fp, st))
        e[2].record()
        torch.cuda.synchronize()
        k2.append(e[0].elapsed_time(e[1]))
        k3.append(e[1].elapsed_time(e[2]))
    out[name] = {"k2_us": 1e3 * sum(k2) / len(k2), "k3_us": 1e3 * sum(k3) / len(k3)}
    eng.close()
print(json.dumps({"size": [w, h], **out}))
