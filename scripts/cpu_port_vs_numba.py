"""CPU baseline translation (build container only: needs /root/reference):
the reference's own numba engine (pkg/src/rgbdseg/engine.py, workers = all
threads) beside the oracle C port (oracle/, what bench.py's cpu_baseline and
--impl reference time on the GPU box) on the same 1920x1080 frames, GMM 7/3
(regime S) + PBAS n=20 (regime T) per frame, after a burn-in.  Prints one
JSON line: Mpixel/s of each and port/numba."""
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from rgbdseg.config import PipelineConfig as RefConfig  # noqa: E402
from rgbdseg.engine import SegmentationEngine as RefEngine  # noqa: E402
from rgbdseg.gmm import GmmParams as RefGmm  # noqa: E402
from rgbdseg.pbas import PbasParams as RefPbas  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2002_00250_b200 import synth  # noqa: E402
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig  # noqa: E402

W, H = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (1920, 1080)))
threads = oracle.cpu_threads()
fs = [synth.make_frame("S", W, H, 0, t) for t in range(7)]
ft = [synth.make_frame("T", W, H, 0, t) for t in range(7)]


def run(make, workers, budget=20.0, burn=22):
    g = make("gmm", workers)
    p = make("pbas", workers)
    for t in range(burn):
        g.process_frame(fs[t % 7])
        p.process_frame(ft[t % 7])
    n, el = 0, 0.0
    while el < budget or n < 2:
        t0 = time.perf_counter()
        g.process_frame(fs[n % 7])
        p.process_frame(ft[n % 7])
        el += time.perf_counter() - t0
        n += 1
    return W * H * n / el / 1e6, n


def ref_make(algo, workers):
    cfg = RefConfig(algorithm=algo, mode="rgbd", workers=workers, seed=1,
                    gmm=RefGmm(k_rgb=7, k_d=3), pbas=RefPbas(n=20))
    return RefEngine(cfg, W, H)


def port_make(algo, workers):
    cfg = PipelineConfig(algorithm=algo, mode="rgbd", seed=1, gmm=GmmParams(k_rgb=7, k_d=3),
                         pbas=PbasParams(n=20))
    return oracle.OracleEngine(cfg, W, H, workers=workers)


out = {"width": W, "height": H, "threads": threads, "cpu": open("/proc/cpuinfo").read().split(
    "model name")[1].split("\n")[0].strip(" \t:")}
for tag, mk in (("numba", ref_make), ("port", port_make)):
    out[f"{tag}_mpix_s"], out[f"{tag}_frames"] = run(mk, threads)
    out[f"{tag}_mpix_s_1thread"], _ = run(mk, 1, budget=10.0, burn=22)
out["port_over_numba"] = out["port_mpix_s"] / out["numba_mpix_s"]
out["port_over_numba_1thread"] = out["port_mpix_s_1thread"] / out["numba_mpix_s_1thread"]
print(json.dumps(out))
