"""pixel_rng / rng_stream evaluated by the DEVICE twin of the counter-based
generator (engine_rng.py:55-64) -- the very __device__ functions the PBAS
kernel inlines (csrc/common.cuh), exposed so tests can pin them against the
reference's values (tests/test_rng.py:15-21)."""

from __future__ import annotations

import numpy as np

from . import _native
from .engine import default_device

_M64 = (1 << 64) - 1


def pixel_keys(keys: np.ndarray, device: int | None = None) -> np.ndarray:
    """keys: (N, 5) uint64 (seed, x, y, frame, draw) -> (N,) f64 draws."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1, 5)
    out = np.empty(len(keys), dtype=np.float64)
    dev = default_device() if device is None else device
    rc = _native.lib().rgbdseg_rng_keys(keys.ctypes.data, len(keys), out.ctypes.data, dev)
    _native.check(rc, "rng_keys")
    return out


def pixel_rng(seed, x, y, frame_idx, draw_idx, device: int | None = None) -> float:
    """Uniform draw in [0, 1), a pure function of its five arguments."""
    k = np.array([[int(v) & _M64 for v in (seed, x, y, frame_idx, draw_idx)]], dtype=np.uint64)
    return float(pixel_keys(k, device)[0])


def rng_stream(seed, x, y, frame_idx, count, device: int | None = None) -> np.ndarray:
    """count consecutive draws at one pixel."""
    out = np.empty(int(count), dtype=np.float64)
    dev = default_device() if device is None else device
    rc = _native.lib().rgbdseg_rng_stream(int(seed) & _M64, int(x) & _M64, int(y) & _M64,
                                          int(frame_idx) & _M64, int(count), out.ctypes.data, dev)
    _native.check(rc, "rng_stream")
    return out
