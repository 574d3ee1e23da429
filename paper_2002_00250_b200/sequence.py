"""Whole-sequence driver: the reference's `process_sequence` / `RunStats`
(pkg/src/rgbdseg/engine.py:32-45, :146-214) on the device path.

Per frame: depth resampled to the RGB size when they differ, packed and
segmented -- all three on the GPU (`SegmentationEngine.apply`, frames.py:
46-88 fused into one staging kernel) -- and the mask returned to the host.
The timing covers resample + pack + segment + the mask read-back, as the
reference's does (disk I/O excluded).  With `labels`, every frame's
confusion counts are accumulated inside K1/K2 (metrics.compare_masks fused)
and the pooled report (aggregate_sequence) comes back in `stats.report`.

Sources: any object with `__len__`, `frame_id(i)` and `load(i) -> (rgb,
depth16 or None)` (e.g. `MemorySequence`); a reference `SequenceSource`
(rgb_paths / depth_paths) is read through the reference's own frame_io when
that package is importable -- file I/O is not part of this package.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .errors import SequenceError


@dataclass
class RunStats:
    """Segment-stage timing for a run (engine.py:32-45); disk I/O excluded."""

    frames_processed: int = 0
    seconds: float = 0.0
    per_frame_seconds: list = field(default_factory=list)
    report: Optional[object] = None  # metrics.MetricsReport when labels were given

    @property
    def fps(self) -> float:
        return self.frames_processed / self.seconds if self.seconds > 0 else float("inf")

    @property
    def seconds_per_frame(self) -> float:
        return self.seconds / self.frames_processed if self.frames_processed else 0.0


class MemorySequence:
    """In-memory frame source: rgb (H, W, 3) uint8 frames, optional 16-bit
    depth maps (any size; resampled on the device) and frame ids."""

    def __init__(self, rgb, depth16=None, ids=None):
        self.rgb = list(rgb)
        self.depth16 = None if depth16 is None else list(depth16)
        if self.depth16 is not None and len(self.depth16) != len(self.rgb):
            raise SequenceError("rgb and depth sequences differ in length")
        self.ids = list(ids) if ids is not None else [f"{i:06d}" for i in range(len(self.rgb))]
        self.depth_paths = self.depth16  # the reference's "has depth" test (engine.py:162)

    def __len__(self) -> int:
        return len(self.rgb)

    def frame_id(self, i: int) -> str:
        return self.ids[i]

    def load(self, i: int):
        return self.rgb[i], (None if self.depth16 is None else self.depth16[i])


def _loader(source):
    if hasattr(source, "load"):
        return source.load
    try:  # a reference SequenceSource on disk: read it with the reference's own I/O
        from rgbdseg import frames as frame_io  # the reference engine.py:23 alias
    except ImportError as exc:  # pragma: no cover - depends on the caller's environment
        raise SequenceError("source has no load(i) and rgbdseg.frames is not importable") from exc

    def load(i):
        rgb = frame_io.load_rgb(source.rgb_paths[i])
        d = frame_io.load_depth(source.depth_paths[i]) if source.depth_paths is not None else None
        return rgb, d

    return load


def process_sequence(source, config, on_mask: Optional[Callable] = None, labels=None,
                     device: Optional[int] = None) -> RunStats:
    """Run a whole sequence through the engine (engine.py:146-214).

    on_mask(frame_id, mask) receives every (H, W) uint8 mask; labels, when
    given, is a sequence of per-frame ground truths (arrays of 0 bg / 1 fg /
    2 ignore, or GroundTruthMask objects) -- stats.report then holds the
    pooled PWC / FNR / FPR / Si."""
    from .engine import SegmentationEngine
    from .metrics import aggregate_sequence

    if len(source) == 0:
        raise SequenceError("sequence is empty")
    use_depth = config.mode == "rgbd"
    if use_depth and getattr(source, "depth_paths", None) is None:
        raise SequenceError("rgbd mode needs a depth directory")
    if labels is not None and len(labels) != len(source):
        raise SequenceError("labels must cover every frame of the sequence")
    load = _loader(source)
    out_dir, write_png = None, None
    if getattr(config, "emit_masks", False):  # engine.py:165-171; PNG writing is the reference's
        if config.out_dir is None:
            raise SequenceError("emit_masks is set but no out_dir configured")
        try:
            from rgbdseg import frames as frame_io  # noqa: PLC0415
        except ImportError as exc:
            raise SequenceError("emit_masks needs the reference's rgbdseg.frames (PNG I/O)") from exc
        from pathlib import Path

        out_dir = Path(config.out_dir)
        out_dir.mkdir(parents=True, exist_ok=True)
        write_png = frame_io.write_mask_png
    stats = RunStats()
    engine = None
    try:
        for i in range(len(source)):
            try:
                rgb, depth16 = load(i)
            except Exception as exc:
                raise SequenceError(f"frame {i} ({source.frame_id(i)}): {exc}") from exc
            rgb = np.asarray(rgb)
            if engine is None:
                engine = SegmentationEngine(config, rgb.shape[1], rgb.shape[0], device)
            elif (rgb.shape[0], rgb.shape[1]) != (engine.height, engine.width):
                raise SequenceError(
                    f"frame {i} ({source.frame_id(i)}): dimensions {rgb.shape[1]}x{rgb.shape[0]} "
                    f"differ from sequence {engine.width}x{engine.height}")
            t0 = time.perf_counter()
            frame = engine.pack(rgb, depth16 if use_depth else None)
            if labels is not None:
                mask = engine.process_frame(frame, labels=labels[i])
            else:
                mask = engine.process_frame(frame)
            mask = mask.cpu().numpy()
            dt = time.perf_counter() - t0
            stats.frames_processed += 1
            stats.seconds += dt
            stats.per_frame_seconds.append(dt)
            if out_dir is not None:
                write_png(out_dir / f"{source.frame_id(i)}.png", mask)
            if on_mask is not None:
                on_mask(source.frame_id(i), mask)
        if labels is not None:
            stats.report = aggregate_sequence([engine.confusion_counts()])
    finally:
        if engine is not None:
            engine.close()
    return stats
