"""Plugin-level drop-in: the reference's per-algorithm state objects
(`GmmState`, pkg/src/rgbdseg/gmm.py:230-280; `PbasState`, pbas.py:279-337)
backed by the B200 handles, for a host that keeps the reference's own
`SegmentationEngine` (engine.py:53-143) and swaps only the model grids:

    # rgbdseg/engine.py, inside SegmentationEngine.__init__
    from paper_2002_00250_b200.plugin import GmmStateB200 as GmmState, PbasStateB200 as PbasState

The reference engine splits every frame into `workers` row bands
(engine.py:48-50) and calls `segment_rows` once per band -- concurrently on
a thread pool when workers > 1 (engine.py:114-124, :126-143) -- and, for
PBAS, `apply_intents` once per band afterwards.  The device segments a whole
frame in one launch, so:

  * the FIRST band call of a frame runs the whole frame (classification,
    and for PBAS the race-free intent application) and writes the whole
    mask; every further band call of that frame finds its rows written and
    returns (concurrent callers wait on a lock until the frame is done);
  * PBAS `segment_rows` returns 0 intents and `apply_intents` is a no-op:
    the device already applied them, after every pixel classified
    (pbas.py:511-522 semantics);
  * a new frame starts when a band's rows were already covered in the
    current frame (GMM: calls carry no frame index) or when the frame index
    changes (PBAS); empty bands (more workers than rows) are harmless.

`arrays()` is a live mapping in the reference layout from construction on,
as the reference's (tests/test_acceptance.py:125-139 takes it before the
first frame and reads it after every frame).  Errors are the reference's
exception classes (errors.py).
"""

from __future__ import annotations

import threading
from collections.abc import Mapping

import numpy as np

from .config import PipelineConfig
from .errors import ConfigError


class _Covered:
    """Row ranges of the current frame that band calls have claimed."""

    def __init__(self, height: int):
        self.height = int(height)
        self.ranges: list = []

    def full(self) -> bool:
        return sum(y1 - y0 for y0, y1 in self.ranges) >= self.height

    def overlaps(self, y0: int, y1: int) -> bool:
        return any(y0 < b1 and b0 < y1 for b0, b1 in self.ranges)


class _LiveArrays(Mapping):
    """arrays(): always reads the owner's current device state (the handle may
    be re-created before the first frame, when the first band call brings
    the depth mode / seed the constructor does not see)."""

    def __init__(self, owner):
        self._owner = owner

    def _view(self):
        return self._owner._current().state_arrays()

    def __getitem__(self, key):
        return self._view()[key]

    def __iter__(self):
        return iter(self._view())

    def __len__(self):
        return len(self._view())


class _DeviceState:
    def __init__(self, width: int, height: int, device=None):
        self.width, self.height = int(width), int(height)
        self.device = device
        self.engine = None
        self._cfg = None
        self._frames = 0  # frames segmented by the current handle
        self._lock = threading.Lock()
        self._cov = _Covered(height)

    def _default_config(self) -> PipelineConfig:
        raise NotImplementedError

    def _ensure(self, cfg: PipelineConfig):
        """The handle for `cfg`; before the first frame a handle created for
        another depth mode / seed (state still initial) is replaced."""
        from .engine import SegmentationEngine

        key = (cfg.mode, cfg.seed)
        if self.engine is not None and self._cfg != key:
            if self._frames:
                raise ConfigError("the depth mode / seed changed after the first frame")
            self.engine.close()
            self.engine = None
        if self.engine is None:
            self.engine = SegmentationEngine(cfg, self.width, self.height, device=self.device)
            self._cfg = key
        return self.engine

    def _current(self):
        with self._lock:
            return self.engine if self.engine is not None else self._ensure(self._default_config())

    def arrays(self):
        """Live mapping in the reference layout (gmm.py:251-255 / pbas.py:296-303),
        valid from construction on, as the reference's."""
        return _LiveArrays(self)

    def close(self) -> None:
        if self.engine is not None:
            self.engine.close()
            self.engine = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GmmStateB200(_DeviceState):
    """GmmState (gmm.py:230-280): GmmStateB200(width, height, params)."""

    def __init__(self, width: int, height: int, params, device=None):
        params.validate()
        super().__init__(width, height, device)
        self.params = params

    def segment_rows(self, frame: np.ndarray, y0: int, y1: int, use_depth: bool,
                     mask: np.ndarray) -> None:
        """gmm.py:272-280; rows [y0, y1) of `mask` hold the decisions on return."""
        if y1 <= y0:  # empty band
            return
        with self._lock:
            new_frame = not self._cov.ranges or self._cov.full() or self._cov.overlaps(y0, y1)
            if not new_frame:  # another band of a frame already segmented
                self._cov.ranges.append((y0, y1))
                return
            eng = self._ensure(PipelineConfig(algorithm="gmm",
                                              mode="rgbd" if use_depth else "rgb_only",
                                              gmm=self.params))
            np.copyto(mask, eng.process_frame(frame))
            self._frames += 1
            self._cov.ranges = [(y0, y1)]

    def _default_config(self) -> PipelineConfig:
        return PipelineConfig(algorithm="gmm", mode="rgbd", gmm=self.params)


class PbasStateB200(_DeviceState):
    """PbasState (pbas.py:279-337): PbasStateB200(width, height, params).
    The seed arrives with every band call (engine.py:127-128); the handle is
    created at the first call (its per-column RNG table depends on it)."""

    def __init__(self, width: int, height: int, params, device=None):
        params.validate()
        super().__init__(width, height, device)
        self.params = params
        self._frame = None
        self._seed = None

    def segment_rows(self, frame: np.ndarray, frame_idx: int, y0: int, y1: int, use_depth: bool,
                     seed, mask: np.ndarray, intents: np.ndarray) -> int:
        """pbas.py:320-333; returns the number of intents left for
        apply_intents -- always 0, the device applied them itself."""
        if y1 <= y0:
            return 0
        with self._lock:
            if self._frame == int(frame_idx) and not self._cov.overlaps(y0, y1):
                self._cov.ranges.append((y0, y1))
                return 0
            if self._frames and int(seed) != self._seed:
                raise ConfigError("the seed changed between frames of one PbasState")
            self._seed = int(seed)
            eng = self._ensure(PipelineConfig(algorithm="pbas",
                                              mode="rgbd" if use_depth else "rgb_only",
                                              pbas=self.params, seed=int(seed)))
            if eng.frame_idx != int(frame_idx):  # the caller's frame index is authoritative
                eng.frame_idx = int(frame_idx)
            np.copyto(mask, eng.process_frame(frame))
            self._frames += 1
            self._frame = int(frame_idx)
            self._cov.ranges = [(y0, y1)]
            return 0

    def _default_config(self) -> PipelineConfig:
        return PipelineConfig(algorithm="pbas", mode="rgbd", pbas=self.params, seed=0)

    def apply_intents(self, frame: np.ndarray, intents: np.ndarray, count: int,
                      use_depth: bool) -> None:
        """pbas.py:335-337: nothing left to apply (count is always 0)."""
        if count:
            raise ConfigError("PbasStateB200 never hands out intents")
