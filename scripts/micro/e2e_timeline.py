"""Timeline of the shared-upload e2e pipeline (MultiCameraPipeline schedule,
8 x 1080p, GMM 7/3 + PBAS n=20): CUDA events around every copy-in, compute
and copy-out of 12 steps; prints per-step start/end (ms) per stream, plus
copy-only and compute-only step rates."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import _gen_ring  # noqa: E402
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig  # noqa: E402
from paper_2002_00250_b200.engine import MultiStreamEngine  # noqa: E402

w, h, S = 1920, 1080, 8
npix = w * h
dev = torch.device("cuda", 0)
engs = {"gmm": MultiStreamEngine(PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=7, k_d=3)),
                                 w, h, S, device=0),
        "pbas": MultiStreamEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20)),
                                  w, h, S, device=0)}
R = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ring = torch.from_numpy(_gen_ring("T", w, h, list(range(S)), R)).to(dev)  # (S, R, H, W, 4)
pinned = torch.empty((R, S, h, w, 4), dtype=torch.uint8, pin_memory=True)
pinned.copy_(ring.transpose(0, 1))
D = 2
dframes = torch.empty((D, S, h, w, 4), dtype=torch.uint8, device=dev)
dmasks = {k: torch.empty((D, S, h, w), dtype=torch.uint8, device=dev) for k in engs}
hmask = {k: [torch.empty((S, h, w), dtype=torch.uint8, pin_memory=True) for _ in range(D)] for k in engs}
s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
s_c = {k: torch.cuda.Stream(dev) for k in engs}
BURN = int(sys.argv[1]) if len(sys.argv) > 1 else 60
for t in range(BURN):  # burn-in
    for k, e in engs.items():
        fb = ring.data_ptr()
        e.step_ptrs([fb + ((i * R) + t % R) * npix * 4 for i in range(S)],
                    [dmasks[k].data_ptr() + i * npix for i in range(S)], s_c[k].cuda_stream)
torch.cuda.synchronize()


def E():
    return torch.cuda.Event(enable_timing=True)


def run(n, copy_in=True, compute=True, copy_out=True, log=None):
    free = [None] * D
    t0 = E()
    t0.record(s_in)
    for q in (s_out, *s_c.values()):
        q.wait_event(t0)
    for t in range(n):
        k = t % D
        rec = {}
        if free[k] is not None:
            s_in.wait_event(free[k])
        a, b = E(), E()
        a.record(s_in)
        if copy_in:
            with torch.cuda.stream(s_in):
                dframes[k].copy_(pinned[t % R], non_blocking=True)
        b.record(s_in)
        rec["in"] = (a, b)
        for name, e in engs.items():
            st = s_c[name]
            st.wait_event(b)
            a2, b2 = E(), E()
            a2.record(st)
            if compute:
                fb = dframes[k].data_ptr()
                e.step_ptrs([fb + i * npix * 4 for i in range(S)],
                            [dmasks[name][k].data_ptr() + i * npix for i in range(S)], st.cuda_stream)
            b2.record(st)
            rec[name] = (a2, b2)
            s_out.wait_event(b2)
        a3, b3 = E(), E()
        a3.record(s_out)
        if copy_out:
            with torch.cuda.stream(s_out):
                for name in engs:
                    hmask[name][k].copy_(dmasks[name][k], non_blocking=True)
        b3.record(s_out)
        rec["out"] = (a3, b3)
        free[k] = b3
        if log is not None:
            log.append(rec)
    torch.cuda.synchronize()
    return t0


res = {}
for tag, kw in (("all", {}), ("no_copies", {"copy_in": False, "copy_out": False}),
                ("copies_only", {"compute": False}), ("no_copy_out", {"copy_out": False})):
    run(3, **kw)
    h0 = time.perf_counter()
    run(30, **kw)
    res[tag + "_ms_per_step"] = (time.perf_counter() - h0) / 30 * 1e3
log = []
t0 = run(8, log=log)
res["timeline"] = [{k: [round(t0.elapsed_time(a), 3), round(t0.elapsed_time(b), 3)] for k, (a, b) in r.items()}
                   for r in log]
print(json.dumps(res))

from paper_2002_00250_b200.pipeline import MultiCameraPipeline  # noqa: E402

pipe = MultiCameraPipeline({}, w, h, S, device=0, engines=engs)
hout = [{k: torch.empty((S, h, w), dtype=torch.uint8, pin_memory=True) for k in engs} for _ in range(2)]
for t in range(3):
    pipe.submit(pinned[t % R], hout[t % 2])
pipe.synchronize()
sub = 0.0
h0 = time.perf_counter()
for t in range(30):
    a = time.perf_counter()
    pipe.submit(pinned[t % R], hout[t % 2])
    sub += time.perf_counter() - a
pipe.synchronize()
res2 = {"pipeline_ms_per_step": (time.perf_counter() - h0) / 30 * 1e3, "pipeline_submit_host_ms": sub / 30 * 1e3}
print(json.dumps(res2))
