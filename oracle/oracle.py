"""ctypes front end of the C restatement (oracle/rgbdseg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.

`OracleEngine` mirrors the reference `SegmentationEngine`
(pkg/src/rgbdseg/engine.py:53-143): the state lives in numpy arrays in the
reference layout (gmm.py:244-249, pbas.py:285-294) and `process_frame`
runs one frame over `workers` row bands exactly as the reference engine does.
`pixel_rng_py` is the pure-int twin of tests/reference.py:28-41.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle_rgbdseg.so"
_lib = None

_MASK64 = (1 << 64) - 1


def build() -> Path:
    """Compile the restatement with oracle/Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    L = ctypes.CDLL(str(_LIB_PATH))
    u64, i64, i32, f64 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    vp = ctypes.c_void_p
    L.oracle_pixel_rng.restype = f64
    L.oracle_pixel_rng.argtypes = [u64, u64, u64, u64, u64]
    L.oracle_rng_stream.restype = None
    L.oracle_rng_stream.argtypes = [u64, u64, u64, u64, i64, vp]
    L.oracle_gmm_band.restype = None
    L.oracle_gmm_band.argtypes = [i64, i64, vp, i64, i64] + [vp] * 6 + [i32, i32] + [f64] * 6 + [i32, vp]
    L.oracle_gmm_frame.restype = ctypes.c_int
    L.oracle_gmm_frame.argtypes = [i64, i64, vp] + [vp] * 6 + [i32, i32] + [f64] * 6 + [i32, vp, i32]
    L.oracle_pbas_band.restype = i64
    L.oracle_pbas_band.argtypes = ([i64, i64, vp, i64, i64, i64] + [vp] * 10 + [u64, i32, i32]
                                   + [f64] * 7 + [i32, vp, vp])
    L.oracle_pbas_band_emit.restype = i64
    L.oracle_pbas_band_emit.argtypes = ([i64, i64, vp, i64, i64, i64] + [vp] * 10 + [u64, i32, i32]
                                        + [f64] * 7 + [i32, vp, vp, vp])
    L.oracle_pbas_frame.restype = i64
    L.oracle_pbas_frame.argtypes = ([i64, i64, vp, i64] + [vp] * 10 + [u64, i32, i32]
                                    + [f64] * 7 + [i32, vp, i32])
    L.oracle_pbas_frame_g.restype = i64
    L.oracle_pbas_frame_g.argtypes = ([i64, i64, vp, i64] + [vp] * 10 + [u64, i32, i32]
                                      + [f64] * 7 + [i32, vp, i32, vp, vp, f64, f64, vp])
    L.oracle_pbas_gradient_weight.restype = ctypes.c_uint32
    L.oracle_pbas_gradient_weight.argtypes = [u64, i64, f64, f64]
    L.oracle_pbas_gradient_map.restype = u64
    L.oracle_pbas_gradient_map.argtypes = [i64, i64, vp, vp]
    L.oracle_pbas_apply_intents.restype = None
    L.oracle_pbas_apply_intents.argtypes = [i64, i32, vp, vp, vp, i64, i32]
    _lib = L
    return L


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def pixel_rng(seed, x, y, frame_idx, draw_idx) -> float:
    """engine_rng.py:36-44 restated in C."""
    return lib().oracle_pixel_rng(seed & _MASK64, x & _MASK64, y & _MASK64,
                                  frame_idx & _MASK64, draw_idx & _MASK64)


def rng_stream(seed, x, y, frame_idx, count) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    lib().oracle_rng_stream(seed & _MASK64, x, y, frame_idx, count, _p(out))
    return out


def _mix64_py(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def pixel_rng_py(seed: int, x: int, y: int, frame_idx: int, draw_idx: int) -> float:
    """Pure-int twin (reference tests/reference.py:34-41)."""
    h = (seed ^ 0x5851F42D4C957F2D) & _MASK64
    h = _mix64_py(h ^ ((x * 0x9E3779B97F4A7C15) & _MASK64))
    h = _mix64_py(h ^ ((y * 0xC2B2AE3D27D4EB4F) & _MASK64))
    h = _mix64_py(h ^ ((frame_idx * 0x165667B19E3779F9) & _MASK64))
    h = _mix64_py(h ^ ((draw_idx * 0xD6E8FEB86659FD93) & _MASK64))
    return (h >> 11) * 2.0 ** -53


def gmm_state(width, height, params) -> dict:
    """GmmState.__init__ (gmm.py:238-249)."""
    k, kd = params.k_rgb, params.k_d
    return {
        "rgb_w": np.zeros((height, width, k)),
        "rgb_mu": np.zeros((height, width, k, 3)),
        "rgb_var": np.full((height, width, k), float(params.var_init)),
        "d_w": np.zeros((height, width, kd)),
        "d_mu": np.zeros((height, width, kd, 1)),
        "d_var": np.full((height, width, kd), float(params.var_init)),
    }


def pbas_state(width, height, params) -> dict:
    """PbasState.__init__ (pbas.py:279-294)."""
    n = params.n
    return {
        "samples": np.zeros((height, width, n, 4), dtype=np.uint8),
        "dmin_rgb": np.zeros((height, width, n), dtype=np.uint8),
        "dmin_d": np.zeros((height, width, n), dtype=np.uint8),
        "len_rgb": np.zeros((height, width), dtype=np.uint8),
        "pos_rgb": np.zeros((height, width), dtype=np.uint8),
        "len_d": np.zeros((height, width), dtype=np.uint8),
        "pos_d": np.zeros((height, width), dtype=np.uint8),
        "r_rgb": np.full((height, width), float(params.r_init)),
        "r_d": np.full((height, width), float(params.r_init)),
        "t": np.full((height, width), float(params.t_init)),
    }


class OracleEngine:
    """CPU twin of the reference SegmentationEngine (engine.py:53-143).

    `config` is any object with the PipelineConfig fields (algorithm, mode,
    gmm, pbas, seed, workers); the package's own PipelineConfig qualifies.
    """

    def __init__(self, config, width: int, height: int, workers: int | None = None):
        self.config = config
        self.width = width
        self.height = height
        self.frame_idx = 0
        self.use_depth = config.mode == "rgbd"
        self.workers = workers if workers is not None else getattr(config, "workers", 1)
        self.gradient = None
        # opt-in f32 GMM storage (package extension, csrc/gmm.cu StF32): every
        # stored value rounded to nearest f32 -- rounding the whole state after
        # each frame is the same rule, since pixels are independent and values
        # the frame did not touch are already f32-representable
        self.gmm_f32 = getattr(config, "gmm_state_dtype", "float64") == "float32"
        if config.algorithm == "gmm":
            self.state = gmm_state(width, height, config.gmm)
            self._round_f32()
        else:
            self.state = pbas_state(width, height, config.pbas)
            self.gradient = getattr(config, "pbas_gradient", None)
            if self.gradient is not None:  # opt-in feature, see oracle_pbas_frame_g
                self.state["samples_grad"] = np.zeros((height, width, config.pbas.n), np.uint8)
                self.state["grad_prev_sum"] = np.full((), GRAD_NONE, dtype=np.uint64)

    def state_arrays(self) -> dict:
        return self.state

    def _round_f32(self):
        if self.gmm_f32:
            for v in self.state.values():
                v[...] = v.astype(np.float32).astype(np.float64)

    def process_frame(self, frame: np.ndarray) -> np.ndarray:
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        assert frame.shape == (self.height, self.width, 4), frame.shape
        mask = np.empty((self.height, self.width), dtype=np.uint8)
        L = lib()
        st = self.state
        if self.config.algorithm == "gmm":
            p = self.config.gmm
            rc = L.oracle_gmm_frame(
                self.width, self.height, _p(frame),
                _p(st["rgb_w"]), _p(st["rgb_mu"]), _p(st["rgb_var"]),
                _p(st["d_w"]), _p(st["d_mu"]), _p(st["d_var"]),
                p.k_rgb, p.k_d, p.alpha, p.s, p.tau, p.match_lambda * p.match_lambda,
                p.var_init, p.w_init, int(self.use_depth), _p(mask), self.workers)
            assert rc == 0
            self._round_f32()
        else:
            p = self.config.pbas
            args = (self.width, self.height, _p(frame), self.frame_idx,
                    _p(st["samples"]), _p(st["dmin_rgb"]), _p(st["dmin_d"]),
                    _p(st["len_rgb"]), _p(st["pos_rgb"]), _p(st["len_d"]), _p(st["pos_d"]),
                    _p(st["r_rgb"]), _p(st["r_d"]), _p(st["t"]),
                    int(self.config.seed) & _MASK64, p.n, p.min_matches,
                    p.r_lower, p.r_scale, p.r_inc_dec, p.t_lower, p.t_upper, p.t_inc, p.t_dec,
                    int(self.use_depth), _p(mask), self.workers)
            if self.gradient is None:
                rc = L.oracle_pbas_frame(*args)
            else:
                g = self.gradient
                rc = L.oracle_pbas_frame_g(*args, _p(st["samples_grad"]), _p(st["grad_prev_sum"]),
                                           float(g.alpha), float(g.mean_init), None)
            assert rc >= 0
        self.frame_idx += 1
        return mask

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def pbas_band_emit(cfg, state, frame, frame_idx, y0, y1, mask):
    """One PBAS row band with global coordinates (pbas.py:344-508); returns
    (intents (k,3) = (ny, nx, slot), emitters (k,2) = (y, x)) in emission order."""
    h, w = frame.shape[:2]
    p = cfg.pbas
    cap = max((y1 - y0) * w, 1)
    intents = np.empty((cap, 3), dtype=np.int64)
    emitters = np.empty((cap, 2), dtype=np.int64)
    st = state
    k = lib().oracle_pbas_band_emit(
        w, h, _p(frame), frame_idx, y0, y1,
        _p(st["samples"]), _p(st["dmin_rgb"]), _p(st["dmin_d"]),
        _p(st["len_rgb"]), _p(st["pos_rgb"]), _p(st["len_d"]), _p(st["pos_d"]),
        _p(st["r_rgb"]), _p(st["r_d"]), _p(st["t"]),
        int(cfg.seed) & _MASK64, p.n, p.min_matches,
        p.r_lower, p.r_scale, p.r_inc_dec, p.t_lower, p.t_upper, p.t_inc, p.t_dec,
        int(cfg.mode == "rgbd"), _p(mask), _p(intents), _p(emitters))
    return intents[:k], emitters[:k]


GRAD_NONE = (1 << 64) - 1  # grad_prev_sum before the first frame: use mean_init


def gradient_map(frame: np.ndarray) -> tuple[np.ndarray, int]:
    """Opt-in gradient feature's magnitude map (oracle_pbas_gradient_map)."""
    frame = np.ascontiguousarray(frame, dtype=np.uint8)
    h, w = frame.shape[:2]
    g = np.empty((h, w), dtype=np.uint8)
    total = lib().oracle_pbas_gradient_map(w, h, _p(frame), _p(g))
    return g, int(total)


def gradient_weight(prev_sum: int, npix: int, alpha: float, mean_init: float) -> int:
    return int(lib().oracle_pbas_gradient_weight(prev_sum, npix, alpha, mean_init))


def gradient_map_np(frame: np.ndarray) -> np.ndarray:
    """Independent numpy statement of the same map: 3x3 Sobel per channel on
    an edge-replicated frame, L1 magnitude, max over r,g,b, >> 3."""
    f = np.pad(frame[:, :, :3].astype(np.int64), ((1, 1), (1, 1), (0, 0)), mode="edge")
    h, w = frame.shape[:2]

    def at(dy, dx):
        return f[1 + dy:1 + dy + h, 1 + dx:1 + dx + w]

    sx = (at(-1, 1) + 2 * at(0, 1) + at(1, 1)) - (at(-1, -1) + 2 * at(0, -1) + at(1, -1))
    sy = (at(1, -1) + 2 * at(1, 0) + at(1, 1)) - (at(-1, -1) + 2 * at(-1, 0) + at(-1, 1))
    return ((np.abs(sx) + np.abs(sy)).max(axis=2) >> 3).astype(np.uint8)


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def scale_depth_map(depth16: np.ndarray) -> np.ndarray:
    """frames.scale_depth_map (frames.py:46-52), numpy restatement."""
    d = depth16.astype(np.uint32)
    d8 = np.maximum((d * 255) // 65535, 1)
    d8[depth16 == 0] = 0
    return d8.astype(np.uint8)


def resample_depth(depth16: np.ndarray, target_w: int, target_h: int) -> np.ndarray:
    """frames.resample_depth (frames.py:73-88): nearest neighbour on pixel centres, f64 index."""
    src_h, src_w = depth16.shape
    if (src_w, src_h) == (target_w, target_h):
        return depth16.copy()
    ys = np.minimum(((np.arange(target_h) + 0.5) * src_h / target_h).astype(np.int64), src_h - 1)
    xs = np.minimum(((np.arange(target_w) + 0.5) * src_w / target_w).astype(np.int64), src_w - 1)
    return depth16[np.ix_(ys, xs)]


def pack_frame(rgb: np.ndarray, depth16: np.ndarray | None) -> np.ndarray:
    """frames.pack_frame (frames.py:55-70) after resampling depth to the RGB size."""
    h, w = rgb.shape[:2]
    frame = np.zeros((h, w, 4), dtype=np.uint8)
    frame[:, :, :3] = rgb
    if depth16 is not None:
        frame[:, :, 3] = scale_depth_map(resample_depth(depth16, w, h))
    return frame


def compare_masks(result: np.ndarray, labels: np.ndarray):
    """metrics.compare_masks (metrics.py:50-69): (tp, tn, fp, fn); label 2 = ignore."""
    fg = result > 127
    gt_fg, gt_bg = labels == 1, labels == 0
    return (int(np.count_nonzero(fg & gt_fg)), int(np.count_nonzero(~fg & gt_bg)),
            int(np.count_nonzero(fg & gt_bg)), int(np.count_nonzero(~fg & gt_fg)))


def median3x3(mask: np.ndarray) -> np.ndarray:
    """Opt-in postprocess oracle: scipy.ndimage.median_filter(size=3, mode='reflect')."""
    from scipy import ndimage

    return ndimage.median_filter(mask, size=3, mode="reflect")
