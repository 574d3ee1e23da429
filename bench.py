#!/usr/bin/env python
"""Throughput benchmark of the B200 RGB-D segmentation path.

Metric (BASELINE.json): "Mpixel/s and fps at 1920x1080 RGB-D (GMM, PBAS),
1/2/4/8 B200, % HBM roofline".

Default workload = BASELINE config 4 at its per-GPU share: 8 independent
1920x1080 RGB-D camera streams per GPU (64 on 8 GPUs), every frame segmented
by BOTH the GMM (paper default k_rgb=7, k_d=3) and PBAS (n=20).
One step = one frame of every stream of this rank through both algorithms:
one batched GMM launch + one batched PBAS classify launch + one batched PBAS
apply launch.  `value` = whole-job Mpixel/s (pixels of all streams of all
ranks per second, each pixel segmented by both algorithms); weak scaling
(per-GPU work fixed as N grows).

Inputs: SURVEY.md §8(d) regimes, generated untimed and uploaded to HBM as a
frame ring per stream: GMM runs on regime S (every component seeded, so the
algorithmic byte count is honest), PBAS on regime T (moving objects + depth
holes).  The state is burned in before anything is timed: GMM 8 frames (all
7/3 components seeded); PBAS --pbas-age frames (default 400), because its
work per frame grows with model age (update probability 1/T, T adapting down
to t_lower after ~300 frames) -- the timed window and the PBAS
per_algo/roofline are at steady state (model_age: T median = t_lower), and
frames 40-90 of the burn-in (young model, PBAS alone) are reported as
`pbas_young`.  The per-step working set (5.8 GB GMM + 2.5 GB PBAS state per
GPU) is far larger than L2, so no explicit flush is needed; smaller
workloads (configs 1-2) flush L2 between individually timed steps.

Extra keys: roofline (GMM K1, the dominant kernel), per-algorithm breakdown,
cpu_baseline (the oracle port on this host's cores), e2e (the public
host-buffer APIs with H2D/D2H inside the timed region: MultiCameraPipeline
with one shared upload per camera frame, and e2e.dropin = the reference's
per-frame SegmentationEngine.process_frame(numpy) call on one stream),
clocks (nvidia-smi sampled during the timed region), gpu_launches.

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port of the numba kernels, oracle/, all host threads) on the same
workload, one 1080p stream-frame (GMM + PBAS) per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2002_00250_b200 import synth  # noqa: E402
from paper_2002_00250_b200.config import (GmmParams, PbasGradient, PbasParams,  # noqa: E402
                                          PipelineConfig)

METRIC = "Mpixel/s and fps at 1920x1080 RGB-D (GMM, PBAS), 1/2/4/8 B200, % HBM roofline"
UNIT = "Mpixel/s"
# SURVEY.md §8(d) algorithmic bytes per pixel per frame (B_alg).
B_ALG = {("gmm", 7, 3): 485, ("gmm", 3, 3): 293, ("pbas", 20): 181,
         # opt-in gradient feature (--pbas-gradient): + n bytes of per-sample magnitudes read
         ("pbas_grad", 20): 201,
         # opt-in f32 GMM state storage (--gmm-state f32)
         ("gmm_f32", 7, 3): 245, ("gmm_f32", 3, 3): 149}

WORKLOADS = {
    # name: (width, height, streams per GPU, gmm (k_rgb, k_d) or None, pbas n or None)
    "config4": (1920, 1080, 8, (7, 3), 20),
    "config3": (1280, 720, 1, (7, 3), 20),
    "config1": (640, 480, 1, (3, 3), None),
    "config2": (640, 480, 1, None, 20),
    # one 7680x4320 frame split into row bands, one per GPU (PBAS n=20)
    "config5": (7680, 4320, 1, None, 20),
}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """SM clocks + throttle reasons sampled every 2 ms through NVML (a polling
    thread, so even a ~0.2 s warm-up + timed region gets ~100 samples);
    falls back to `nvidia-smi -lms 50` when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int, pci_bus_id: str | None = None):
        self.gpu = gpu_index
        self.pci = pci_bus_id
        self.proc = None
        self.f = None
        self.thread = None
        self.samples = []

    def _nvml_start(self) -> bool:
        try:
            import threading

            import pynvml as nv

            nv.nvmlInit()
            h = None
            if self.pci and "RGBDSEG_NVSMI_INDEX" not in os.environ:
                try:
                    h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
                except Exception:
                    h = None
            if h is None:
                h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        except Exception:
            return False
        self._stop = threading.Event()

        def poll():
            while not self._stop.is_set():
                try:
                    mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((mhz, max_mhz, {n for n, b in zip(self.NAMES, bits) if r & b}))
                except Exception:
                    pass
                self._stop.wait(0.002)

        self.thread = threading.Thread(target=poll, daemon=True)
        self.thread.start()
        return True

    def start(self):
        if self._nvml_start():
            return
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.gpu)],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=5)
            rows = self.samples
            src = "nvml"
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.flush()
            rows = []
            for ln in Path(self.f.name).read_text().splitlines():
                r = ln.split(",")
                try:
                    rows.append((float(r[1]), float(r[2]),
                                 {n for n, v in zip(self.NAMES, r[4:8]) if v.strip().lower() == "active"}))
                except (ValueError, IndexError):
                    continue
            os.unlink(self.f.name)
            src = "nvidia-smi"
        else:
            return None
        if not rows:
            return None
        reasons = set().union(*(r[2] for r in rows))
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows), "source": src}


def _throttled(clock_info, dev, world) -> bool:
    """hw_slowdown / hw_thermal_slowdown / sw_thermal_slowdown seen on any rank
    (sw_power_cap is kept and noted)."""
    bad = bool(clock_info and set(clock_info["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                                            "sw_thermal_slowdown"})
    if world > 1:
        import torch
        import torch.distributed as dist

        flag = torch.tensor([int(bad)], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        bad = bool(flag.item())
    return bad


def _pci_bus_id(dev) -> str | None:
    try:
        p = torch.cuda.get_device_properties(dev)
        return f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        return None


# --------------------------------------------------------------- frames ---
def _gen_ring(regime, w, h, seeds, ring, k_rgb=7):
    jobs = [(s, t) for s in seeds for t in range(ring)]
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        frames = list(ex.map(lambda st: synth.make_frame(regime, w, h, st[0], st[1], k_rgb), jobs))
    return np.stack(frames).reshape(len(seeds), ring, h, w, 4)


# --------------------------------------------------------- bit equality ----
def _fold_dev(t) -> int:
    """Position-weighted 64-bit fold of a device tensor's bytes (wrapping
    int64 arithmetic): equal bytes at equal positions <=> equal folds, up to
    2^-64 collisions.  Used to prove a row-band / multi-rank run equals the
    single-band one without moving the data."""
    import torch

    b = t.contiguous().view(torch.uint8).flatten()
    pad = (-b.numel()) % 8
    if pad:
        b = torch.cat([b, torch.zeros(pad, dtype=torch.uint8, device=b.device)])
    words = b.view(torch.int64)
    idx = torch.arange(words.numel(), device=words.device, dtype=torch.int64) * 2 + 1
    return int((words * idx).sum().item())


def _fold_np(a) -> int:
    b = np.ascontiguousarray(a).view(np.uint8).ravel()
    pad = (-b.size) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    words = b.view(np.uint64)
    idx = np.arange(words.size, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    with np.errstate(over="ignore"):
        return int((words * idx).sum(dtype=np.uint64))


def _mix(acc: int, v: int) -> int:
    return ((acc * 0x9E3779B97F4A7C15) ^ (v & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF


# --------------------------------------------------------- CPU baseline ----
def _native_k2_mode(ms_engine) -> int:
    from paper_2002_00250_b200 import _native

    return int(_native.lib().rgbdseg_pbas_get_k2_mode(ms_engine.engines[0]._h.ptr))


def _k2_name(ms_engine) -> str:
    return {1: "rows", 2: "strips", 3: "fused K2+K3 (one cooperative launch)"}.get(
        _native_k2_mode(ms_engine), "?")


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_sample(w, h, gmm_k, pbas_n, seed, budget_s=12.0, max_frames=400, workers=None):
    """Time the oracle port (reference algorithm, CPU) on a bounded sample:
    one w x h stream, GMM + PBAS per frame, after an untimed burn-in."""
    from oracle import oracle

    oracle.build()
    workers = workers or oracle.cpu_threads()
    engines = []
    if gmm_k:
        g = oracle.OracleEngine(PipelineConfig(algorithm="gmm", mode="rgbd",
                                               gmm=GmmParams(k_rgb=gmm_k[0], k_d=gmm_k[1])),
                                w, h, workers=workers)
        engines.append((g, "S", 8))
    if pbas_n:
        p = oracle.OracleEngine(PipelineConfig(algorithm="pbas", mode="rgbd",
                                               pbas=PbasParams(n=pbas_n), seed=seed + 1),
                                w, h, workers=workers)
        engines.append((p, "T", pbas_n + 2))
    ring = {r: [synth.make_frame(r, w, h, seed, t, gmm_k[0] if gmm_k else 7) for t in range(7)]
            for r in {e[1] for e in engines}}
    for eng, reg, burn in engines:
        for t in range(burn):
            eng.process_frame(ring[reg][t % 7])
    frames, elapsed = 0, 0.0
    while frames < max_frames and (elapsed < budget_s or frames < 2):
        t0 = time.perf_counter()
        for eng, reg, _ in engines:
            eng.process_frame(ring[reg][frames % 7])
        elapsed += time.perf_counter() - t0
        frames += 1
    return {"value": w * h * frames / elapsed / 1e6, "unit": UNIT, "cores": workers,
            "kind": "port", "frames": frames, "seconds": elapsed,
            "sample": f"{frames} frames of one {w}x{h} stream through "
                      f"{'GMM %d/%d' % gmm_k if gmm_k else ''}"
                      f"{' + ' if gmm_k and pbas_n else ''}{'PBAS n=%d' % pbas_n if pbas_n else ''}"
                      f" (oracle/ C port of the numba kernels, {workers} threads, after burn-in)"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    w, h, _, gmm_k, pbas_n = WORKLOADS[args.workload]
    from oracle import oracle

    oracle.build()
    workers = oracle.cpu_threads()
    engines = []
    if gmm_k:
        engines.append((oracle.OracleEngine(
            PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=gmm_k[0], k_d=gmm_k[1])),
            w, h, workers=workers), "S", 8))
    if pbas_n:
        engines.append((oracle.OracleEngine(
            PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=pbas_n), seed=1),
            w, h, workers=workers), "T", pbas_n + 2))
    ring = {r: [synth.make_frame(r, w, h, 0, t, gmm_k[0] if gmm_k else 7) for t in range(7)]
            for r in {e[1] for e in engines}}
    for eng, reg, burn in engines:
        for t in range(burn):
            eng.process_frame(ring[reg][t % 7])

    def step(i):
        for eng, reg, _ in engines:
            eng.process_frame(ring[reg][i % 7])

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = w * h * args.steps / dt / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64/u8", "data": "synthetic",
        "config": {"workload": f"{args.workload}: reference CPU path, one {w}x{h} RGB-D stream-frame "
                               f"per step", "width": w, "height": h,
                   "gmm": list(gmm_k) if gmm_k else None, "pbas_n": pbas_n},
        "fps": args.steps / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "cpu_model": _cpu_model(),
                         "sample": f"{args.steps} timed steps x one {w}x{h} frame (GMM+PBAS), "
                                   f"oracle/ C port of the reference numba kernels, {workers} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm ---
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2002_00250_b200.engine import MultiStreamEngine

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w, h, S, gmm_k, pbas_n = WORKLOADS[args.workload]
    if args.streams:
        S = args.streams
    npix = w * h
    stream_ids = [rank * S + i for i in range(S)]  # global stream ids (content seeds)

    # ---- engines + device frame rings (untimed setup)
    algos = []
    if gmm_k:
        gcfg = PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=gmm_k[0], k_d=gmm_k[1]),
                              gmm_state_dtype="float32" if args.gmm_state == "f32" else "float64")
        g = MultiStreamEngine(gcfg, w, h, S, device=local_rank, seeds=[s + 1 for s in stream_ids])
        ring_s = torch.from_numpy(_gen_ring("S", w, h, stream_ids, gmm_k[0], gmm_k[0])).to(dev)
        algos.append(("gmm", g, ring_s,
                      B_ALG.get(("gmm_f32" if args.gmm_state == "f32" else "gmm",) + tuple(gmm_k))))
    if pbas_n:
        pcfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=pbas_n),
                              pbas_gradient=PbasGradient() if args.pbas_gradient else None)
        p = MultiStreamEngine(pcfg, w, h, S, device=local_rank, seeds=[s + 1 for s in stream_ids])
        if args.k2_mode != "auto":  # pin the K2 variant (evidence runs; results are identical)
            from paper_2002_00250_b200 import _native

            for e in p.engines:
                _native.check(_native.lib().rgbdseg_pbas_set_k2_mode(
                    e._h.ptr, {"rows": 1, "strips": 2, "fused": 3, "unfused": 4}[args.k2_mode]),
                    "set_k2_mode")
        ring_t = torch.from_numpy(_gen_ring("T", w, h, stream_ids, 8)).to(dev)
        algos.append(("pbas", p, ring_t,
                      B_ALG.get(("pbas_grad" if args.pbas_gradient else "pbas", pbas_n))))
    # One CUDA stream and one mask buffer per algorithm: GMM (HBM-bound) and
    # PBAS (latency-bound K3) are independent engines and run concurrently.
    # PBAS (latency-bound) on a higher-priority stream: the block scheduler
    # then interleaves its blocks with the bandwidth-bound GMM blocks instead
    # of draining the whole GMM grid first (--stream-priority 0 disables).
    prio = {"pbas": -args.stream_priority, "gmm": 0}
    streams = {a[0]: torch.cuda.Stream(dev, priority=prio[a[0]]) for a in algos}
    masks = {a[0]: torch.empty((S, h, w), dtype=torch.uint8, device=dev) for a in algos}
    main = streams[algos[0][0]]
    torch.cuda.set_stream(main)

    def launch(name, eng, ring, t):
        R = ring.shape[1]
        base = ring.data_ptr()
        fptrs = [base + ((i * R) + (t % R)) * npix * 4 for i in range(S)]
        mb = masks[name].data_ptr()
        eng.step_ptrs(fptrs, [mb + i * npix for i in range(S)], streams[name].cuda_stream)

    # Working sets below 4x L2 (configs 1-2: 55-90 MB of state) would be
    # timed warm out of the 126 MB L2: flush L2 between timed steps instead
    # (a 2x-L2 write, outside the events) and time every step separately.
    l2_bytes = getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20)
    state_bytes = sum((a[3] or 0) for a in algos) * npix * S
    flush_buf = (torch.empty(2 * l2_bytes, dtype=torch.uint8, device=dev)
                 if state_bytes < 4 * l2_bytes else None)

    def flush_l2(k):
        # 2x-L2 write (evicts every line of the workload), then -- unless
        # --flush write -- a read pass over the same buffer so the dirty
        # flush lines are written back HERE, untimed, and the timed step
        # starts from a cold but clean L2 (otherwise the step pays the
        # flush's own ~126 MB write-back).
        if flush_buf is not None:
            flush_buf.fill_(k & 0xFF)
            if args.flush == "write+read":
                flush_buf.amax()

    # Burn-in.  GMM: 8 frames seed every component.  PBAS: its per-frame
    # work grows with model age (update probability 1/T, T adapting down to
    # t_lower over ~300 frames of the synthetic scene), so it is
    # aged to steady state (--pbas-age frames, T = t_lower) before anything
    # is timed; frames 40-90 of the burn-in (young model, PBAS alone) are
    # timed on the way and reported as `pbas_young`.
    burn_of = {a[0]: (8 if a[0] == "gmm" else max(2 * pbas_n, args.pbas_age)) for a in algos}
    burn = max(burn_of.values())
    young = None
    yw = (2 * pbas_n, 2 * pbas_n + 50) if pbas_n else None
    ev_y = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
    young_pairs = []  # small configs: every young frame timed alone after an L2 flush
    for t in range(burn):
        in_young = bool(yw and "pbas" in streams and burn_of["pbas"] >= yw[1])
        if in_young and flush_buf is None and t in yw:
            ev_y[yw.index(t)].record(streams["pbas"])
        if in_young and t == yw[1]:
            torch.cuda.synchronize()
            pe = next(a[1] for a in algos if a[0] == "pbas")
            tt = pe.engines[0].state_arrays()["t"]
            ms_y = (ev_y[0].elapsed_time(ev_y[1]) / (yw[1] - yw[0]) if flush_buf is None else
                    statistics.mean(a.elapsed_time(b) for a, b in young_pairs))
            young = {"frames": list(yw), "pbas_T_median": float(np.median(tt)),
                     "ms_per_step": ms_y, "k2_variant": _k2_name(pe),
                     "l2": "inputs larger than L2" if flush_buf is None else "L2 flushed per frame"}
        timed_young = in_young and flush_buf is not None and yw[0] <= t < yw[1]
        for name, eng, ring, _ in algos:
            if t < burn_of[name]:
                if timed_young and name == "pbas":
                    with torch.cuda.stream(streams[name]):
                        flush_l2(t)
                    pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    pair[0].record(streams[name])
                    launch(name, eng, ring, t)
                    pair[1].record(streams[name])
                    young_pairs.append(pair)
                else:
                    launch(name, eng, ring, t)
    torch.cuda.synchronize()
    t_frame_by = dict(burn_of)

    # ---- solo phase: each algorithm alone, per-launch CUDA events on its own
    # stream -> the per-kernel durations the roofline is computed from.
    launches_per_step = sum(1 if a[0] == "gmm" else 2 for a in algos)
    solo = max(10, min(args.steps, 50))
    per_algo_ms = {}
    for name, eng, ring, _ in algos:
        st = streams[name]
        t_frame = t_frame_by[name]
        if flush_buf is None:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(solo + 1)]
            for k in range(solo):
                evs[k].record(st)
                launch(name, eng, ring, t_frame)
                t_frame += 1
            evs[solo].record(st)
            torch.cuda.synchronize()
            per_algo_ms[name] = [evs[k].elapsed_time(evs[k + 1]) for k in range(solo)]
        else:  # cold L2 for every launch: flush, then an event pair per launch
            pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(solo)]
            with torch.cuda.stream(st):
                for k in range(solo):
                    flush_l2(k)
                    pairs[k][0].record(st)
                    launch(name, eng, ring, t_frame)
                    pairs[k][1].record(st)
                    t_frame += 1
            torch.cuda.synchronize()
            per_algo_ms[name] = [a.elapsed_time(b) for a, b in pairs]
        t_frame_by[name] = t_frame

    # ---- warm-up + timed region (concurrent schedule)
    def step():
        for name, eng, ring, _ in algos:
            launch(name, eng, ring, t_frame_by[name])
            t_frame_by[name] += 1

    remeasured = False
    for attempt in range(2):  # a throttled run (hw/thermal slowdown) is re-measured once
        clocks = ClockSampler(int(os.environ.get("RGBDSEG_NVSMI_INDEX", local_rank)), _pci_bus_id(dev))
        clocks.start()  # sampling spans warm-up + timed region (both under full load)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        def timed(n):
            """n steps between one event pair (fork/join of the algorithm streams)."""
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(main)
            for name in streams:
                if streams[name] is not main:
                    streams[name].wait_event(start)
            for _ in range(n):
                step()
            for name in streams:
                if streams[name] is not main:
                    done = torch.cuda.Event()
                    done.record(streams[name])
                    main.wait_event(done)
            end.record(main)
            return start, end

        if flush_buf is None:
            spans = [timed(args.steps)]
        else:  # cold L2 every step: flush on main (untimed), then one timed step
            spans = []
            for k in range(args.steps):
                flush_l2(k)
                spans.append(timed(1))
        torch.cuda.synchronize()
        clock_info = clocks.stop()
        if attempt == 0 and _throttled(clock_info, dev, world):
            remeasured = True
            continue
        break
    if world > 1:
        dist.barrier()
    elapsed_ms = sum(a.elapsed_time(b) for a, b in spans)

    # ---- final metric reduction (NCCL all-reduce of counters, once per run)
    fg = sum(torch.count_nonzero(m) for m in masks.values()).to(torch.int64)
    counters = torch.stack([fg, torch.tensor(sum(m.numel() for m in masks.values()), device=dev,
                                             dtype=torch.int64)])
    t_max = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(counters, op=dist.ReduceOp.SUM)
    elapsed_ms = float(t_max.item())
    ms_step = elapsed_ms / args.steps
    total_px = npix * S * world * args.steps
    value = total_px / (elapsed_ms / 1e3) / 1e6
    fps = S * world * args.steps / (elapsed_ms / 1e3)

    peak, peak_kind = measured_peaks()
    per_algo = {}
    for name, eng, ring, balg in algos:
        avg_ms = statistics.mean(per_algo_ms[name])
        mpx = npix * S / (avg_ms / 1e3) / 1e6
        d = {"ms_per_step": avg_ms, "mpix_s_per_gpu": mpx, "fps_per_stream": 1e3 / avg_ms,
             "bytes_per_pixel_alg": balg}
        if balg:
            gbs = balg * npix * S / (avg_ms / 1e3) / 1e9
            d.update({"achieved_gbs": gbs, "roofline_frac": gbs / peak})
        per_algo[name] = d
    dom = "gmm" if "gmm" in per_algo else "pbas"
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            tkey = dom + ("_f32" if dom == "gmm" and args.gmm_state == "f32" else
                          "_grad" if dom == "pbas" and args.pbas_gradient else "")
            traffic = json.loads(tfile.read_text()).get(f"{tkey}:{args.workload}")
        except Exception:
            traffic = None
    # PBAS's measured bytes per launch at the steady state the bench times
    # (strip K2 + K3 list, ncu), beside its algorithmic bytes
    if "pbas" in per_algo and tfile.exists() and not args.pbas_gradient:
        try:
            tj = json.loads(tfile.read_text())
            k2, k3 = tj.get(f"pbas:{args.workload}"), tj.get(f"pbas_apply:{args.workload}")
            if k2 is not None and k3 is not None:
                per_algo["pbas"]["traffic_per_step_ncu"] = k2 + k3
                per_algo["pbas"]["traffic_frac_of_peak"] = (
                    (k2 + k3) / (per_algo["pbas"]["ms_per_step"] / 1e3) / 1e9 / peak)
        except Exception:
            pass
    roof = {"bound": "hbm", "achieved": per_algo[dom].get("achieved_gbs"), "peak": peak,
            "unit": "GB/s", "frac": per_algo[dom].get("roofline_frac"), "traffic": traffic,
            "kernel": (f"gmm_step_kernel<{gmm_k[0]},{gmm_k[1]},{'StF32' if args.gmm_state == 'f32' else 'StF64'}> (K1)"
                       if dom == "gmm" else "pbas_classify_kernel (K2)"),
            "peak_kind": peak_kind,
            "bytes_per_launch_alg": (per_algo[dom]["bytes_per_pixel_alg"] or 0) * npix * S}

    # PBAS's per-frame work grows with model age (update probability 1/T, T
    # adapting down): report the timed frame window and T then.
    age_info = {}
    for name, eng, _, _ in algos:
        done = t_frame_by[name]  # frames this engine has segmented
        age_info[f"{name}_timed_frames"] = [done - args.steps, done]
        age_info[f"{name}_solo_frames"] = [done - args.steps - args.warmup - solo,
                                           done - args.steps - args.warmup]
        if name == "pbas":
            tt = eng.engines[0].state_arrays()["t"]
            age_info.update({"pbas_T_median": float(np.median(tt)),
                             "pbas_T_at_t_lower": float(np.mean(tt == eng.config.pbas.t_lower)),
                             "pbas_k2_variant": _k2_name(eng)})
    if young is not None:
        peak_y, _ = measured_peaks()
        balg = B_ALG.get(("pbas_grad" if args.pbas_gradient else "pbas", pbas_n))
        gbs = balg * npix * S / (young["ms_per_step"] / 1e3) / 1e9
        young.update({"achieved_gbs": gbs, "roofline_frac": gbs / peak_y})

    # ---- per-stream digests (untimed): a stream's result depends only on its
    # global id (content seed, PBAS seed), never on how many GPUs share the
    # job, so stream g's digest must be identical in the N = 1, 2, 4, 8 runs
    digests = None
    if not args.no_verify:
        mine = {}
        for i, g in enumerate(stream_ids):
            acc = 0
            for name, eng, _, _ in algos:
                acc = _mix(acc, _fold_dev(masks[name][i]))
                st_i = eng.engines[i].state_arrays()
                acc = _mix(acc, _fold_np(st_i["rgb_w" if name == "gmm" else "samples"]))
            mine[g] = f"{acc:016x}"
        if world > 1:
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            digests = {k: v for d in allv for k, v in d.items()}
        else:
            digests = mine

    # ---- e2e through the public host-buffer API (rank-local, then max)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, algos, S, w, h, dev, world)

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(w, h, gmm_k, pbas_n, seed=0, budget_s=args.cpu_budget)
            # also one core, and name the CPU
            one = cpu_sample(w, h, gmm_k, pbas_n, seed=0, budget_s=max(2.0, args.cpu_budget / 4),
                             max_frames=40, workers=1)
            cpu["value_1_core"] = one["value"]
            cpu["sample_1_core"] = one["sample"]
            cpu["cpu_model"] = _cpu_model()
        except Exception as exc:  # report, never fail the bench line
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        wl_desc = (f"{args.workload}: {S} x {w}x{h} RGB-D streams per GPU"
                   + (f", GMM {gmm_k[0]}/{gmm_k[1]} (regime S)" if gmm_k else "")
                   + (f", PBAS n={pbas_n} (regime T)" if pbas_n else "")
                   + (" with the opt-in gradient feature (not the reference algorithm)"
                      if pbas_n and args.pbas_gradient else "")
                   + (" with opt-in f32 GMM state storage (north_star tolerance, not bit parity)"
                      if gmm_k and args.gmm_state == "f32" else ""))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (f32 GMM state)/u8" if gmm_k and args.gmm_state == "f32" else "f64/u8",
            "data": "synthetic (SURVEY.md §8(d) regimes S/T, seeded per stream)",
            "config": {"workload": wl_desc, "width": w, "height": h, "streams_per_gpu": S,
                       "streams_total": S * world,
                       "gmm": list(gmm_k) if gmm_k else None, "pbas_n": pbas_n,
                       "gmm_state": args.gmm_state if gmm_k else None,
                       "pbas_gradient": ({"alpha": PbasGradient().alpha,
                                          "mean_init": PbasGradient().mean_init}
                                         if args.pbas_gradient else None),
                       "burn_in_frames": burn_of,
                       "l2": (f"inputs larger than L2 (state per step {state_bytes / 1e9:.2f} GB "
                              f">> {l2_bytes >> 20} MB)" if flush_buf is None else
                              f"L2 flushed between timed steps ({2 * l2_bytes >> 20} MB {args.flush}, "
                              f"untimed; state per step {state_bytes / 1e6:.0f} MB < 4x L2), "
                              "each step timed by its own event pair"),
                       "parallelism": f"streams sharded {S}/GPU over {world} GPU(s)",
                       "schedule": "GMM and PBAS engines on two CUDA streams, concurrently "
                                   f"(PBAS priority +{args.stream_priority}); per_algo/roofline "
                                   "from a solo phase of each right before the timed window "
                                   "(same model age: PBAS at steady state, T = t_lower)"},
            "fps": fps,
            "per_algo": per_algo,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": (dict(clock_info, remeasured=remeasured) if clock_info else None),
            "fg_fraction_last_step": float(counters[0].item()) / float(counters[1].item()),
            "model_age": age_info,
            "pbas_young": young,
            "stream_digests": digests,
            "stream_digest_check": ("per global stream id: 64-bit folds of its last GMM and PBAS "
                                    "masks, GMM rgb_w and PBAS samples after the run; a stream's "
                                    "digest must not depend on the GPU count"),
            "ranks": world,
        }
        print(json.dumps(line), flush=True)
    for _, eng, _, _ in algos:
        eng.close()
    return 0


def run_config5(args, rank, world, local_rank):
    """BASELINE config 5: PBAS on one 7680x4320 stream, row bands across the
    ranks (engine.py:48-50 split), one-row intent halo per frame through
    peer-memory mailboxes (bands.RowBandPbas, csrc/peer.cu; --halo nccl for
    the NCCL send/recv variant).  value = Mpixel/s of the whole frame."""
    import torch
    import torch.distributed as dist

    from paper_2002_00250_b200.bands import RowBandPbas

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w, h, _, _, n = WORKLOADS["config5"]
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=n), seed=1)
    band = RowBandPbas(cfg, w, h, rank, world, device=local_rank, transport=args.halo)
    y0, y1 = band.y0, band.y1
    ring = torch.from_numpy(_gen_ring("T", w, h, [0], 4)[0][:, y0:y1].copy()).to(dev)
    mask = torch.empty((y1 - y0, w), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    t = 0
    acc = 0  # fold of this band's mask, every untimed frame (bit-equality proof)
    for _ in range(2 * n):  # burn-in: warm-up fill + full dmin rings
        band.step(ring[t % 4], mask)
        acc = _mix(acc, _fold_dev(mask))
        t += 1
    clocks = ClockSampler(int(os.environ.get("RGBDSEG_NVSMI_INDEX", local_rank)), _pci_bus_id(dev))
    clocks.start()  # sampling spans warm-up + timed region (both under full load)
    for _ in range(args.warmup):  # BASELINE config 5 is a 60-frame sequence: stay young
        band.step(ring[t % 4], mask)
        acc = _mix(acc, _fold_dev(mask))
        t += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        band.step(ring[t % 4], mask)
        t += 1
    end.record(stream)
    torch.cuda.synchronize()
    clock_info = clocks.stop()
    ms = torch.tensor([start.elapsed_time(end)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    elapsed_ms = float(ms.item())
    # ---- bit-equality proof (untimed): this band's mask folds over the
    # untimed frames, its last mask and its final state, gathered on rank 0
    # and compared with a one-band run of the same frames on rank 0's GPU
    mine = [acc, _fold_dev(mask)]
    if band.engine is not None:
        stt = band.engine.state_arrays()
        mine += [_fold_np(stt[k]) for k in sorted(stt)]
    bit_equal = None
    if world > 1 and not args.no_verify:
        allv = [None] * world
        dist.all_gather_object(allv, (y0, y1, mine))
        if rank == 0:
            from paper_2002_00250_b200.bands import band_bounds
            from paper_2002_00250_b200.engine import SegmentationEngine

            full = torch.from_numpy(_gen_ring("T", w, h, [0], 4)[0]).to(dev)
            fm = torch.empty((h, w), dtype=torch.uint8, device=dev)
            bounds = band_bounds(h, world)
            accs = [0] * world
            with SegmentationEngine(cfg, w, h, device=local_rank) as one:
                for k in range(t):
                    one.step_device(full[k % 4].data_ptr(), fm.data_ptr(),
                                    torch.cuda.current_stream(dev).cuda_stream)
                    if k < t - args.steps:
                        accs = [_mix(a, _fold_dev(fm[b0:b1])) for a, (b0, b1) in zip(accs, bounds)]
                ost = one.state_arrays()
                ost = {k: ost[k] for k in sorted(ost)}
                want = []
                for r, (b0, b1) in enumerate(bounds):
                    wv = [accs[r], _fold_dev(fm[b0:b1])]
                    if b1 > b0:
                        wv += [_fold_np(v[b0:b1]) for v in ost.values()]
                    want.append((b0, b1, wv))
            bit_equal = [tuple(x) for x in allv] == want
            del full
    elif world == 1:
        bit_equal = True  # the single band is the reference layout itself
    peak, peak_kind = measured_peaks()
    band_px = (y1 - y0) * w
    achieved = B_ALG[("pbas", n)] * band_px * args.steps / (elapsed_ms / 1e3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": w * h * args.steps / (elapsed_ms / 1e3) / 1e6, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/f64", "data": "synthetic (SURVEY.md §8(d) regime T)",
            "config": {"workload": f"config5: PBAS n={n} on one {w}x{h} RGB-D stream, "
                                   f"{world} row band(s), 1-row intent halo "
                                   f"({'peer-memory mailboxes' if args.halo == 'p2p' else 'NCCL'})",
                       "width": w, "height": h, "bands": world,
                       "l2": "inputs larger than L2 (PBAS state 4.9 GB)",
                       "parallelism": f"row bands x{world} (engine.py:48-50 split)"},
            "fps": args.steps / (elapsed_ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "pbas_classify (K2) + pbas_apply (K3), rank 0 band"},
            "cpu_baseline": None, "e2e": None,
            "model_age": {"timed_frames": [t - args.steps, t],
                          "pbas_T_median": float(__import__("numpy").median(
                              band.engine.state_arrays()["t"])),
                          "pbas_k2_variant": "tiles" if int(__import__(
                              "paper_2002_00250_b200._native", fromlist=["lib"]).lib()
                              .rgbdseg_pbas_get_k2_mode(band.engine._h.ptr)) == 2 else "rows"},
            "gpu_launches": args.steps * (2 if world == 1 else 6),
            "clocks": clock_info,
            "bit_equal_across_gpus": bit_equal,
            "bit_equal_check": ("every band's mask on every untimed frame, its last mask and its "
                                "final state (position-weighted 64-bit folds), gathered from "
                                f"{world} rank(s) and compared with a one-band run of the same "
                                f"{t} frames on rank 0" if world > 1 else "single band"),
            "ranks": world,
            "collective_backend": (dist.get_backend() if world > 1 else None),
        }
        print(json.dumps(line), flush=True)
    band.close()
    return 0


def run_e2e(args, algos, S, w, h, dev, world):
    """The same workload end to end through the public host-buffer APIs,
    H2D of the inputs and D2H of the masks inside the timed region:

      shared   pipeline.MultiCameraPipeline over the burned-in engines: each
               step uploads ONE (S, H, W, 4) batch of camera frames from
               pinned memory, shared by GMM and PBAS (4 B/px in), and
               downloads both masks (2 B/px out); double-buffered so step
               t+1's upload overlaps step t's kernels;
      dropin   SegmentationEngine.process_frame(numpy) -- the reference's
               per-frame call (engine.py:99-112; process_sequence and the
               service use it): one 1920x1080 stream, pageable numpy frame
               in, numpy mask out, GMM engine then PBAS engine per frame
               (each call synchronous, staged through the handle's pinned
               buffers in chunks)."""
    import torch
    import torch.distributed as dist

    from paper_2002_00250_b200.engine import SegmentationEngine
    from paper_2002_00250_b200.pipeline import MultiCameraPipeline

    npix = w * h
    steps = max(3, args.e2e_steps)  # pipeline fill + drain amortised over the steps
    # One camera-frame stream shared by every algorithm (regime T; --e2e-input
    # S for the saturated one).  The PBAS engines are already at steady state
    # on regime T; GMM gets its own engines burned in on the same frames (the
    # bench's GMM state is trained on regime S, and switching the scene under
    # it would time a scene change, not a steady camera).
    src = next((a[2] for a in algos if a[0] == ("gmm" if args.e2e_input == "S" else "pbas")),
               algos[0][2])
    R = src.shape[1]
    engines, owned = {}, []
    for name, eng, ring, _ in algos:
        if ring is src:
            engines[name] = eng
            continue
        from paper_2002_00250_b200.engine import MultiStreamEngine

        fresh = MultiStreamEngine(eng.config, w, h, S, device=dev.index,
                                  seeds=[e.config.seed for e in eng.engines])
        owned.append(fresh)
        engines[name] = fresh
    cs = {name: torch.cuda.Stream(dev) for name in engines}
    dmask = torch.empty((S, h, w), dtype=torch.uint8, device=dev)

    def dev_step(name, t):
        base = src.data_ptr()
        engines[name].step_ptrs([base + ((i * R) + (t % R)) * npix * 4 for i in range(S)],
                                [dmask.data_ptr() + i * npix for i in range(S)], cs[name].cuda_stream)

    for e in owned:  # burn-in of the fresh engines on the shared frames
        name = next(k for k, v in engines.items() if v is e)
        for t in range(50):
            dev_step(name, t)
    torch.cuda.synchronize()
    # device-resident rate on the same shared input (the e2e leg's ceiling)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    first = next(iter(cs.values()))
    ev0.record(first)
    for q in cs.values():
        q.wait_event(ev0)
    for t in range(30):
        for name in engines:
            dev_step(name, t)
    for q in cs.values():
        e_ = torch.cuda.Event()
        e_.record(q)
        first.wait_event(e_)
    ev1.record(first)
    torch.cuda.synchronize()
    dev_ms = ev0.elapsed_time(ev1) / 30
    pipe = MultiCameraPipeline({}, w, h, S, device=dev.index, engines=engines, depth=args.e2e_depth)
    pinned = torch.empty((R, S, h, w, 4), dtype=torch.uint8, pin_memory=True)
    pinned.copy_(src.transpose(0, 1))  # (R, S, H, W, 4): one batch per step
    host_out = [{name: torch.empty((S, h, w), dtype=torch.uint8, pin_memory=True) for name in engines}
                for _ in range(pipe.depth)]

    def step(t):
        return pipe.submit(pinned[t % R], host_out[t % pipe.depth])

    # pinned H2D rate of this box (the leg's other ceiling: 4 B/px in)
    scratch = torch.empty_like(pinned[0], device=dev)
    scratch.copy_(pinned[0], non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(10):
        scratch.copy_(pinned[k % R], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d_gbs = 10 * scratch.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
    del scratch

    for t in range(3):
        step(t)
    pipe.synchronize()
    if world > 1:
        dist.barrier()
    h2d = 0
    t0 = time.perf_counter()
    for t in range(steps):
        h2d = step(3 + t)
    pipe.synchronize()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt = float(tt.item())
    out = {"value": npix * S * world * steps / dt / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": npix * S * len(algos),
           "steps": steps,
           "timing": "host perf_counter from first submit to final synchronize (spans H2D+D2H)",
           "api": "pipeline.MultiCameraPipeline.submit: one shared pinned upload per camera frame "
                  "for all algorithms, double-buffered copy-in / per-algorithm compute / copy-out "
                  "streams",
           "input": f"regime {args.e2e_input} camera frames shared by both algorithms",
           "device_resident_same_input": {
               "ms_per_step": dev_ms, "value": npix * S * world / (dev_ms / 1e3) / 1e6,
               "note": "the same engines and frames with no host copies (the leg's ceiling)"},
           "pcie_h2d_gbs": h2d_gbs,
           "pcie_bound_value": h2d_gbs * 1e9 / 4 * world / 1e6}
    for e in owned:
        e.close()

    # ---- drop-in leg: the reference's per-frame call on one stream
    gmm_k = next((a[1].config.gmm for a in algos if a[0] == "gmm"), None)
    pbas_p = next((a[1].config.pbas for a in algos if a[0] == "pbas"), None)
    engines = []
    if gmm_k is not None:
        engines.append(SegmentationEngine(PipelineConfig(algorithm="gmm", mode="rgbd", gmm=gmm_k),
                                          w, h, device=dev.index))
    if pbas_p is not None:
        engines.append(SegmentationEngine(PipelineConfig(algorithm="pbas", mode="rgbd", pbas=pbas_p,
                                                         seed=1), w, h, device=dev.index))
    frames = [np.ascontiguousarray(src[0, k].cpu().numpy()) for k in range(min(8, src.shape[1]))]
    for t in range(2 * (pbas_p.n if pbas_p else 4) + 5):
        for e in engines:
            e.process_frame(frames[t % len(frames)])
    nd = max(10, args.e2e_steps)
    t0 = time.perf_counter()
    for t in range(nd):
        for e in engines:
            e.process_frame(frames[t % len(frames)])
    dt = time.perf_counter() - t0
    for e in engines:
        e.close()
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt = float(tt.item())
    out["dropin"] = {"value": npix * world * nd / dt / 1e6, "unit": UNIT,
                     "ms_per_frame": dt / nd * 1e3, "frames": nd,
                     "h2d_bytes_per_step": 4 * npix * len(engines),
                     "d2h_bytes_per_step": npix * len(engines),
                     "api": "SegmentationEngine.process_frame(numpy) -> numpy, one stream per rank, "
                            + " then ".join(e.config.algorithm.upper() for e in engines)
                            + " engine per frame (synchronous; pageable numpy in/out)",
                     "timing": "host perf_counter over the frames"}
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="config4")
    ap.add_argument("--streams", type=int, default=0, help="override streams per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gmm-state", choices=["f64", "f32"], default="f64",
                    help="GMM state storage: f64 = the reference's (default, bit parity); "
                         "f32 = opt-in half-width storage (north_star tolerance)")
    ap.add_argument("--flush", choices=["write+read", "write"], default="write+read",
                    help="L2 flush between timed steps of the small configs (1-2)")
    ap.add_argument("--pbas-gradient", action="store_true",
                    help="PBAS with the opt-in gradient feature (K2G; not the reference algorithm)")
    ap.add_argument("--stream-priority", type=int, default=0,
                    help="PBAS stream priority boost over GMM (0 = equal)")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--e2e-depth", type=int, default=3,
                    help="device frame slots of the shared-upload e2e pipeline")
    ap.add_argument("--e2e-input", choices=["T", "S"], default="T",
                    help="camera frames of the shared-upload e2e leg (regime T or S)")
    ap.add_argument("--k2-mode", choices=["auto", "rows", "strips", "fused", "unfused"], default="auto",
                    help="pin PBAS's K2 variant (default: chosen per frame by the update rate)")
    ap.add_argument("--pbas-age", type=int, default=400,
                    help="PBAS burn-in frames before timing (400: T at t_lower, steady state)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the untimed cross-rank bit-equality proof")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--halo", choices=["p2p", "nccl"], default="p2p",
                    help="config5 row-band intent-halo transport")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: several ranks on ONE GPU (gloo plumbing, same device for all)
    # to exercise the multi-rank bench logic on a single-GPU box
    shared = os.environ.get("RGBDSEG_BENCH_SHARED_GPU") == "1"
    if shared:
        local_rank = 0

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.workload == "config5":
            return run_config5(args, rank, world, local_rank)
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
