"""Seeded synthetic RGB-D sequences for parity runs and the benchmark.

Built on the reference's scene vocabulary (pkg/src/rgbdseg/synth.py): the
deterministic textured background `background_rgb` (synth.py:69-80), the
background depth plane 40000 -> 155 (synth.py:36-37), the +90 colour offset
(synth.py:53) and the 80-unit camouflage depth offset (synth.py:52, :144).
The reference scenes carry no noise and no depth holes, so the
two regimes of SURVEY.md §8(d) are generated here:

  regime "T" (typical): background + per-frame noise U{-4..4} (RGB) and
      U{-2..2} (depth), three wrapping moving rectangles of W/6 x H/4 (two
      visible at +90 RGB, one colour-camouflaged at depth 75), i.i.d. 5% depth
      holes plus one persistent hole blob of ~2% of the area.
  regime "S" (saturated): every pixel cycles through K RGB modes (20+33i for
      K=7, 20+100i otherwise) and 3 depth modes (40, 120, 200) from a random
      phase, noise U{-3..3}, 5% holes.  Seeds every GMM component, so the
      GMM roofline is quoted on it.

Every frame is a pure function of (regime, W, H, seed, t); frames are packed
(H, W, 4) uint8 in (r, g, b, d) order (frames.py:46-70 convention).
"""

from __future__ import annotations

import functools

import numpy as np

BG_DEPTH8 = 155          # 40000 * 255 // 65535 (synth.py:36-37 after frames.py:46-52)
CAMO_DEPTH8 = 75         # 155 - depth_offset 80 (synth.py:52)
COLOUR_OFFSET = 90       # synth.py:53


def background_rgb(width: int, height: int) -> np.ndarray:
    """Deterministic textured background (gradients plus hash speckle);
    same construction as the reference synth.background_rgb (synth.py:69-80)."""
    xs = np.arange(width, dtype=np.int64)
    ys = np.arange(height, dtype=np.int64)
    r = 60 + (xs * 120) // max(width - 1, 1)
    g = 60 + (ys * 120) // max(height - 1, 1)
    out = np.empty((height, width, 3), dtype=np.int64)
    out[:, :, 0] = r[None, :]
    out[:, :, 1] = g[:, None]
    out[:, :, 2] = 90 + ((xs[None, :] + ys[:, None]) * 80) // max(width + height - 2, 1)
    speckle = ((xs[None, :] * 73856093) ^ (ys[:, None] * 19349663)) % 17
    return np.clip(out + speckle[:, :, None], 0, 255).astype(np.uint8)


@functools.lru_cache(maxsize=4)
def _background_i16(width: int, height: int) -> np.ndarray:
    """background_rgb as int16, computed once per frame size (read-only)."""
    bg = background_rgb(width, height).astype(np.int16)
    bg.flags.writeable = False
    return bg


def _rects(width: int, height: int, t: int):
    """Three wrapping rectangles (x0, y0, w, h, kind); kind 0 = visible, 1 = camouflaged."""
    rw, rh = max(width // 6, 1), max(height // 4, 1)
    vmax = max(width // 80, 1)
    speeds = (1, max(vmax // 2, 1), vmax)
    rows = (height // 8, (height * 3) // 8, (height * 5) // 8)
    kinds = (0, 1, 0)
    out = []
    for i in range(3):
        x0 = (speeds[i] * t + i * width // 3) % width
        out.append((x0, rows[i], rw, rh, kinds[i]))
    return out


def _paint_wrapped(plane, x0, y0, w, h, fn):
    width = plane.shape[1]
    y1 = min(y0 + h, plane.shape[0])
    x1 = x0 + w
    if x1 <= width:
        fn(plane, slice(y0, y1), slice(x0, x1))
    else:
        fn(plane, slice(y0, y1), slice(x0, width))
        fn(plane, slice(y0, y1), slice(0, x1 - width))


def frame_typical(width: int, height: int, seed: int, t: int) -> np.ndarray:
    """Regime T frame t of stream `seed`."""
    rng = np.random.default_rng([seed, t])
    rgb = _background_i16(width, height).copy()
    depth = np.full((height, width), BG_DEPTH8, dtype=np.int16)
    for x0, y0, w, h, kind in _rects(width, height, t):
        if kind == 0:
            def vis(p, ys, xs):
                p[ys, xs] += COLOUR_OFFSET
            _paint_wrapped(rgb, x0, y0, w, h, vis)
        else:
            def camo(p, ys, xs):
                p[ys, xs] = CAMO_DEPTH8
            _paint_wrapped(depth, x0, y0, w, h, camo)
    rgb += rng.integers(-4, 5, size=rgb.shape, dtype=np.int16)
    depth += rng.integers(-2, 3, size=depth.shape, dtype=np.int16)
    frame = np.empty((height, width, 4), dtype=np.uint8)
    frame[:, :, :3] = np.clip(rgb, 0, 255)
    d = np.clip(depth, 1, 255)
    holes = rng.random((height, width)) < 0.05
    # one persistent blob (~2% of the area) near the lower-right corner
    bh, bw = max(int(height * 0.14), 1), max(int(width * 0.14), 1)
    holes[height - bh - height // 10: height - height // 10, width - bw - width // 10: width - width // 10] = True
    d[holes] = 0
    frame[:, :, 3] = d
    return frame


def saturated_modes(k_rgb: int):
    if k_rgb == 7:
        return [20 + 33 * i for i in range(7)]
    return [20 + (230 // max(k_rgb, 1)) * i if k_rgb > 3 else 20 + 100 * i for i in range(k_rgb)]


def frame_saturated(width: int, height: int, seed: int, t: int, k_rgb: int = 7) -> np.ndarray:
    """Regime S frame t: per-pixel mode cycling."""
    phase = np.random.default_rng([seed, 1 << 20]).integers(0, 1 << 30, size=(height, width))
    rng = np.random.default_rng([seed, t])
    modes = np.asarray(saturated_modes(k_rgb), dtype=np.int16)
    dmodes = np.asarray((40, 120, 200), dtype=np.int16)
    m = (phase + t) % len(modes)
    md = (phase + t) % 3
    frame = np.empty((height, width, 4), dtype=np.uint8)
    base = modes[m]
    noise = rng.integers(-3, 4, size=(height, width, 4), dtype=np.int16)
    for c in range(3):
        frame[:, :, c] = np.clip(base + noise[:, :, c], 0, 255)
    d = np.clip(dmodes[md] + noise[:, :, 3], 1, 255)
    d[rng.random((height, width)) < 0.05] = 0
    frame[:, :, 3] = d
    return frame


def make_frame(regime: str, width: int, height: int, seed: int, t: int, k_rgb: int = 7) -> np.ndarray:
    if regime == "T":
        return frame_typical(width, height, seed, t)
    if regime == "S":
        return frame_saturated(width, height, seed, t, k_rgb)
    raise ValueError(f"unknown regime {regime!r} (expected 'T' or 'S')")


def sequence(regime: str, width: int, height: int, seed: int, frames: int, k_rgb: int = 7):
    return [make_frame(regime, width, height, seed, t, k_rgb) for t in range(frames)]


# ---------------------------------------------------------------------------
# The reference's acceptance scenes (synth.py:38-160), restated so the
# acceptance criteria can run on the device path: every frame is a pure
# function of (spec, t); depth is 16-bit sensor units, GT 0/255.
# ---------------------------------------------------------------------------
BG_DEPTH16 = 40000   # synth.py:36
DEPTH8_UNIT = 257    # synth.py:38


class SceneSpec:
    """SynthSpec (synth.py:41-66) fields used by the scenes below."""

    def __init__(self, scenario, width=160, height=120, frames=160, entry_frame=100,
                 object_w=40, object_h=40, speed=4, depth_offset=80, colour_offset=90):
        self.scenario, self.width, self.height, self.frames = scenario, width, height, frames
        self.entry_frame, self.object_w, self.object_h, self.speed = (entry_frame, object_w,
                                                                      object_h, speed)
        self.depth_offset, self.colour_offset = depth_offset, colour_offset


def scene_rect(spec: SceneSpec, t: int):
    """object_rect (synth.py:83-101)."""
    if spec.scenario in ("static", "illumination_ramp") or t < spec.entry_frame:
        return None
    x0 = 4 + spec.speed * (t - spec.entry_frame)
    if x0 >= spec.width:
        return None
    x1 = min(x0 + spec.object_w, spec.width)
    y0 = max((spec.height - spec.object_h) // 2, 0)
    y1 = min(y0 + spec.object_h, spec.height)
    if x1 <= x0 or y1 <= y0:
        return None
    return x0, y0, x1, y1


def scene_frame(spec: SceneSpec, t: int):
    """(rgb, depth16, gt) at frame t for static / colour_camouflage /
    depth_camouflage (synth.py:104-160)."""
    bg = background_rgb(spec.width, spec.height)
    rect = scene_rect(spec, t)
    rgb = bg
    if spec.scenario == "depth_camouflage" and rect is not None:
        x0, y0, x1, y1 = rect
        rgb = bg.copy()
        region = rgb[y0:y1, x0:x1].astype(np.int32) + spec.colour_offset
        rgb[y0:y1, x0:x1] = np.clip(region, 0, 255).astype(np.uint8)
    depth = np.full((spec.height, spec.width), BG_DEPTH16, dtype=np.uint16)
    gt = np.zeros((spec.height, spec.width), dtype=np.uint8)
    if rect is not None:
        x0, y0, x1, y1 = rect
        if spec.scenario != "depth_camouflage":
            depth[y0:y1, x0:x1] = BG_DEPTH16 - spec.depth_offset * DEPTH8_UNIT
        gt[y0:y1, x0:x1] = 255
    return rgb, depth, gt
