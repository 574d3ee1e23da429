"""Generate the golden fixtures from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package `rgbdseg` from /root/reference/pkg/src and
its test oracle `reference.py` from /root/reference/pkg/tests (read-only; the
numba cache is redirected), runs them on seeded inputs and writes compressed
.npz fixtures next to this script.  Nothing at test time reads
/root/reference: the GPU box only sees these committed files.

Fixtures:
  rng.npz                 pixel_rng over random + extreme keys, rng_stream
                          (engine_rng.py:55-64; tests/test_rng.py:15-21)
  gmm_equiv_<mode>.npz    the reference's own TestKernelEquivalence case
                          (tests/test_gmm.py:223-248) via reference_gmm_run
  pbas_equiv_<mode>.npz   the reference's own TestKernelEquivalence case
                          (tests/test_pbas.py:463-491) via reference_pbas_run
  gmm_<tag>.npz / pbas_<tag>.npz
                          synthetic regime T / S sequences through the
                          reference numba SegmentationEngine (engine.py:60-112),
                          all masks + final state_arrays().
  frames.npz              frames.pack_frame(rgb, resample_depth(d16, W, H))
                          (frames.py:46-88): all 65536 depth values plus
                          up/down/odd mixed-resolution pairs
  accept_c3.npz           acceptance criterion 3 (tests/test_acceptance.py:
                          125-139): 500 noisy 64x64 frames (default_rng(99)),
                          default GMM, workers=2 -- packed masks, per-frame
                          weight-sum / variance extremes, sha256 of the
                          final state
  accept_c7.npz           acceptance criterion 7 (:200-233): the 160x120x200
                          colour_camouflage scene, seed 42, GMM and PBAS,
                          workers 1 -- packed masks, sha256 of every input
                          frame and of the final state
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, str(REPO))

from rgbdseg.config import PipelineConfig  # noqa: E402
from rgbdseg.engine import SegmentationEngine, pixel_rng, rng_stream  # noqa: E402
from rgbdseg.gmm import GmmParams  # noqa: E402
from rgbdseg.pbas import PbasParams  # noqa: E402
from reference import (  # noqa: E402
    gmm_grid_arrays,
    pbas_grid_arrays,
    reference_gmm_run,
    reference_pbas_run,
)

from paper_2002_00250_b200 import synth  # noqa: E402


def _save(name, **arrays):
    path = HERE / name
    np.savez_compressed(path, **arrays)
    print(f"wrote {path.name}: {path.stat().st_size} bytes")


def make_rng():
    rng = np.random.default_rng(0)
    keys = rng.integers(0, 2 ** 20, size=(400, 5), dtype=np.uint64)
    extreme = np.array([
        [2 ** 63 + 11, 1, 2, 3, 4],
        [2 ** 64 - 1, 2 ** 64 - 1, 2 ** 64 - 1, 2 ** 64 - 1, 2],
        [0, 0, 0, 0, 0],
        [1234, 7679, 4319, 999_999, 1],
        [5, 10, 20, 30, 0],
    ], dtype=np.uint64)
    big = rng.integers(0, 2 ** 63, size=(100, 5), dtype=np.uint64)
    keys = np.concatenate([keys, extreme, big])
    values = np.array([pixel_rng(*(int(v) for v in k)) for k in keys])
    stream = rng_stream(42, 17, 23, 0, 4096)
    _save("rng.npz", keys=keys, values=values, stream=stream,
          stream_key=np.array([42, 17, 23, 0], dtype=np.uint64))


def make_gmm_equiv():
    # Verbatim input construction of tests/test_gmm.py:226-237.
    rng = np.random.default_rng(21)
    height, width = 9, 11
    frames = []
    base = rng.integers(0, 200, size=(height, width, 4), dtype=np.uint8)
    for t in range(8):
        f = base.copy()
        f[2:5, t % width] = (250, 250, 250, 200)
        f[:, :, 3][rng.random((height, width)) < 0.2] = 0
        frames.append(f)
    params = GmmParams(k_rgb=3, k_d=2)
    for mode in ("rgbd", "rgb_only"):
        masks, grid = reference_gmm_run(frames, params, mode)
        st = gmm_grid_arrays(grid, params)
        _save(f"gmm_equiv_{mode}.npz", frames=np.stack(frames), masks=np.stack(masks),
              k_rgb=3, k_d=2, **st)


def make_pbas_equiv():
    # Verbatim input construction of tests/test_pbas.py:467-478.
    rng = np.random.default_rng(77)
    height, width = 7, 9
    params = PbasParams(n=5, min_matches=2)
    base = rng.integers(0, 220, size=(height, width, 4), dtype=np.uint8)
    frames = []
    for t in range(14):
        f = base.copy()
        if t >= 7:
            f[3:6, (t * 2) % width] = (255, 255, 255, 30)
        f[:, :, 3][rng.random((height, width)) < 0.25] = 0
        frames.append(f)
    seed = 1234
    for mode in ("rgbd", "rgb_only"):
        masks, grid = reference_pbas_run(frames, params, mode, seed)
        st = pbas_grid_arrays(grid, params)
        _save(f"pbas_equiv_{mode}.npz", frames=np.stack(frames), masks=np.stack(masks),
              n=5, min_matches=2, seed=seed, **st)


def _engine_run(config, frames):
    h, w = frames[0].shape[:2]
    with SegmentationEngine(config, w, h) as eng:
        masks = [eng.process_frame(f).copy() for f in frames]
        st = {k: v.copy() for k, v in eng.state_arrays().items()}
    return np.stack(masks), st


def make_gmm_seq():
    cases = [
        # tag, regime, W, H, frames, k_rgb, k_d, mode, extra params
        ("T73_rgbd", "T", 48, 32, 40, 7, 3, "rgbd", {}),
        ("T33_rgbd", "T", 48, 32, 40, 3, 3, "rgbd", {}),
        ("T33_rgb_only", "T", 48, 32, 40, 3, 3, "rgb_only", {}),
        ("S73_rgbd", "S", 40, 24, 40, 7, 3, "rgbd", {}),
        ("S33_rgbd_tau4", "S", 40, 24, 30, 3, 3, "rgbd", {"tau": 4.0}),
        # small var_init (< VAR_FLOOR) exercises the floor on unseeded slots
        ("T52_varinit05", "T", 24, 16, 20, 5, 2, "rgbd", {"var_init": 0.5, "alpha": 0.05}),
    ]
    for tag, regime, w, h, nf, k, kd, mode, extra in cases:
        frames = synth.sequence(regime, w, h, seed=3, frames=nf, k_rgb=k)
        params = GmmParams(k_rgb=k, k_d=kd, **extra)
        cfg = PipelineConfig(algorithm="gmm", mode=mode, gmm=params, workers=1)
        masks, st = _engine_run(cfg, frames)
        _save(f"gmm_{tag}.npz", frames=np.stack(frames), masks=masks, k_rgb=k, k_d=kd,
              mode=mode, params=np.array([params.alpha, params.s, params.tau, params.match_lambda,
                                          params.var_init, params.w_init]), **st)


def make_pbas_seq():
    cases = [
        ("T20_rgbd", "T", 48, 32, 70, 20, 2, "rgbd", 8, {}),
        ("T20_rgb_only", "T", 48, 32, 60, 20, 2, "rgb_only", 9, {}),
        ("T5_rgbd", "T", 40, 24, 40, 5, 2, "rgbd", 2 ** 63 + 11, {}),
        ("S20_rgbd", "S", 40, 24, 60, 20, 2, "rgbd", 1, {}),
        ("T7_m3", "T", 33, 21, 50, 7, 3, "rgbd", 77,
         {"r_scale": 3.0, "r_inc_dec": 0.1, "t_init": 10.0, "t_lower": 3.0, "t_upper": 40.0}),
    ]
    for tag, regime, w, h, nf, n, mm, mode, seed, extra in cases:
        frames = synth.sequence(regime, w, h, seed=5, frames=nf)
        params = PbasParams(n=n, min_matches=mm, **extra)
        cfg = PipelineConfig(algorithm="pbas", mode=mode, pbas=params, seed=seed, workers=1)
        masks, st = _engine_run(cfg, frames)
        _save(f"pbas_{tag}.npz", frames=np.stack(frames), masks=masks, n=n, min_matches=mm,
              mode=mode, seed=np.uint64(seed),
              params=np.array([params.r_init, params.r_lower, params.r_scale, params.r_inc_dec,
                               params.t_init, params.t_lower, params.t_upper, params.t_inc,
                               params.t_dec]), **st)


def make_frames():
    """frames.pack_frame / scale_depth_map / resample_depth (frames.py:46-88)."""
    from rgbdseg import frames as ref_frames

    rng = np.random.default_rng(11)
    out = {}
    # every 16-bit depth value once (tests/test_frames.py:27-52 is exhaustive too)
    d_all = np.arange(65536, dtype=np.uint16).reshape(256, 256)
    rgb = rng.integers(0, 256, size=(256, 256, 3), dtype=np.uint8)
    out["all_rgb"], out["all_d16"] = rgb, d_all
    out["all_frame"] = ref_frames.pack_frame(rgb, d_all)
    for tag, (w, h), (dw, dh) in (("up", (64, 48), (32, 24)), ("odd", (37, 23), (16, 11)),
                                   ("down", (40, 30), (64, 48)), ("p720_480", (128, 72), (64, 48))):
        rgb = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        d16 = rng.integers(0, 65536, size=(dh, dw), dtype=np.uint16)
        d16[rng.random((dh, dw)) < 0.1] = 0
        out[f"{tag}_rgb"], out[f"{tag}_d16"] = rgb, d16
        out[f"{tag}_frame"] = ref_frames.pack_frame(rgb, ref_frames.resample_depth(d16, w, h))
    _save("frames.npz", **out)


def _sha(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_accept_c3():
    """Criterion 3 (tests/test_acceptance.py:125-139), the reference engine."""
    rng = np.random.default_rng(99)
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd", workers=2)
    masks, wsum_dev, var_min = [], [], []
    with SegmentationEngine(cfg, 64, 64) as eng:
        state = eng.state_arrays()
        for _ in range(500):
            frame = rng.integers(0, 256, size=(64, 64, 4), dtype=np.uint8)
            frame[:, :, 3] = rng.integers(1, 256, size=(64, 64))  # always valid
            masks.append(np.packbits(eng.process_frame(frame) > 0))
            wsum_dev.append(max(float(np.abs(state[k].sum(axis=2) - 1.0).max())
                                for k in ("rgb_w", "d_w")))
            var_min.append(min(float(state[k].min()) for k in ("rgb_var", "d_var")))
        st = {k: v.copy() for k, v in eng.state_arrays().items()}
    _save("accept_c3.npz", masks=np.stack(masks), wsum_dev=np.array(wsum_dev),
          var_min=np.array(var_min), state_keys=np.array(sorted(st)),
          state_sha=np.array([_sha(st[k]) for k in sorted(st)]))


def make_accept_c7():
    """Criterion 7 (tests/test_acceptance.py:200-233): the reference's scene
    frames (synth.rgb_at / depth16_at, what write_sequence stores as PNG,
    lossless) packed by frames.pack_frame, through the reference engine."""
    from rgbdseg import frames as ref_frames
    from rgbdseg.synth import SynthSpec, depth16_at, rgb_at

    spec = SynthSpec(scenario="colour_camouflage", width=160, height=120, frames=200,
                     entry_frame=100)
    frames = [ref_frames.pack_frame(rgb_at(spec, t), depth16_at(spec, t))
              for t in range(spec.frames)]
    out = {"frame_sha": np.array([_sha(f) for f in frames]),
           "rgb_sha": np.array([_sha(rgb_at(spec, t)) for t in range(spec.frames)]),
           "d16_sha": np.array([_sha(depth16_at(spec, t)) for t in range(spec.frames)])}
    for algo in ("gmm", "pbas"):
        cfg = PipelineConfig(algorithm=algo, mode="rgbd", seed=42, workers=1)
        masks, st = _engine_run(cfg, frames)
        out[f"{algo}_masks"] = np.stack([np.packbits(m > 0) for m in masks])
        out[f"{algo}_state_keys"] = np.array(sorted(st))
        out[f"{algo}_state_sha"] = np.array([_sha(st[k]) for k in sorted(st)])
    _save("accept_c7.npz", **out)


MAKERS = {"rng": make_rng, "gmm_equiv": make_gmm_equiv, "pbas_equiv": make_pbas_equiv,
          "gmm_seq": make_gmm_seq, "pbas_seq": make_pbas_seq, "frames": make_frames,
          "accept_c3": make_accept_c3, "accept_c7": make_accept_c7}

if __name__ == "__main__":
    for name in (sys.argv[1:] or MAKERS):
        MAKERS[name]()
