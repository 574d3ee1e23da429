"""Drop-in `SegmentationEngine` on the B200 kernels.

Mirrors the reference engine surface (pkg/src/rgbdseg/engine.py:53-143):
  SegmentationEngine(config, width, height)        engine.py:60-83
  .process_frame(frame) -> mask                    engine.py:99-112
  .state_arrays() -> live dict-like, ref. layout   engine.py:96-97
  .frame_idx / .width / .height / .config / .use_depth
  .close(), context manager                        engine.py:85-94
with the model state resident in HBM (owned by a C-ABI handle, see
include/rgbdseg_b200.h) instead of numpy arrays.

Input/output:
  - numpy (H, W, 4) uint8 frame -> numpy (H, W) uint8 mask (newly allocated),
    through the C-ABI host path (H2D, kernel, D2H on the handle's stream);
  - torch CUDA (H, W, 4) uint8 tensor -> torch CUDA (H, W) uint8 mask, zero
    copy, enqueued on torch's current stream.
Errors: shape mismatch -> DimensionError (engine.py:101-105); config ->
ConfigError; CUDA/runtime -> DeviceError (an RgbdSegError).  No CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from collections.abc import Mapping

import numpy as np

from . import _native
from .config import validate_config
from .errors import ConfigError, DeviceError, DimensionError

_GMM_SHAPES = {
    "rgb_w": lambda h, w, p: ((h, w, p.k_rgb), np.float64),
    "rgb_mu": lambda h, w, p: ((h, w, p.k_rgb, 3), np.float64),
    "rgb_var": lambda h, w, p: ((h, w, p.k_rgb), np.float64),
    "d_w": lambda h, w, p: ((h, w, p.k_d), np.float64),
    "d_mu": lambda h, w, p: ((h, w, p.k_d, 1), np.float64),
    "d_var": lambda h, w, p: ((h, w, p.k_d), np.float64),
}
_PBAS_SHAPES = {
    "samples": lambda h, w, p: ((h, w, p.n, 4), np.uint8),
    "dmin_rgb": lambda h, w, p: ((h, w, p.n), np.uint8),
    "dmin_d": lambda h, w, p: ((h, w, p.n), np.uint8),
    "len_rgb": lambda h, w, p: ((h, w), np.uint8),
    "pos_rgb": lambda h, w, p: ((h, w), np.uint8),
    "len_d": lambda h, w, p: ((h, w), np.uint8),
    "pos_d": lambda h, w, p: ((h, w), np.uint8),
    "r_rgb": lambda h, w, p: ((h, w), np.float64),
    "r_d": lambda h, w, p: ((h, w), np.float64),
    "t": lambda h, w, p: ((h, w), np.float64),
}
# opt-in gradient feature (config.PbasGradient; not in the reference)
_PBAS_GRAD_SHAPES = {
    "samples_grad": lambda h, w, p: ((h, w, p.n), np.uint8),
    "grad_prev_sum": lambda h, w, p: ((), np.uint64),
}


def default_device() -> int:
    """RGBDSEG_DEVICE when set (an explicit override: e.g. every rank of a
    shared-GPU run on one device), else LOCAL_RANK under torchrun, else 0."""
    for var in ("RGBDSEG_DEVICE", "LOCAL_RANK"):
        if var in os.environ:
            return int(os.environ[var])
    return 0


def _is_torch(x) -> bool:
    return type(x).__module__.split(".")[0] == "torch"


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the C-ABI reads a NULL stream as "the handle's own"


def torch_stream_handle(device=None) -> int:
    """cudaStream_t of torch's current stream, as the C-ABI expects it.

    torch reports its default (legacy NULL) stream as 0, which the C-ABI
    would read as "the handle's own stream"; pass cudaStreamLegacy instead
    so the kernels stay ordered with torch's work."""
    import torch

    return torch.cuda.current_stream(device).cuda_stream or CUDA_STREAM_LEGACY


class _Handle:
    """Owns one C-ABI handle (GMM or PBAS)."""

    def __init__(self, algorithm, width, height, params, use_depth, seed, device,
                 band=None, gmm_flags=0):
        L = _native.lib()
        self.L = L
        self.algorithm = algorithm
        self.ptr = ctypes.c_void_p()
        if _native.device_count() <= device:
            raise DeviceError(f"CUDA device {device} not available "
                              f"({_native.device_count()} visible); the B200 path has no CPU fallback")
        if algorithm == "gmm":
            self.pc = _native.gmm_params_c(params)
            rc = L.rgbdseg_gmm_create_ex(width, height, ctypes.byref(self.pc), int(use_depth),
                                         device, gmm_flags, ctypes.byref(self.ptr))
            _native.check(rc, "rgbdseg_gmm_create")
            self.pre = "rgbdseg_gmm_"
        else:
            self.pc = _native.pbas_params_c(params)
            if band is None:
                rc = L.rgbdseg_pbas_create(width, height, ctypes.byref(self.pc), int(use_depth),
                                           int(seed) & ((1 << 64) - 1), device,
                                           ctypes.byref(self.ptr))
            else:
                y0, y1 = band
                rc = L.rgbdseg_pbas_create_band(width, height, y0, y1, ctypes.byref(self.pc),
                                                int(use_depth), int(seed) & ((1 << 64) - 1),
                                                device, ctypes.byref(self.ptr))
            _native.check(rc, "rgbdseg_pbas_create")
            self.pre = "rgbdseg_pbas_"

    def fn(self, name):
        return getattr(self.L, self.pre + name)

    def close(self):
        if self.ptr:
            self.fn("destroy")(self.ptr)
            self.ptr = ctypes.c_void_p()


class StateView(Mapping):
    """Live, read-only view of the device state in the reference layout.

    Each `view[key]` copies the field device->host (and transposes SoA planes
    to (H, W, K[, C]) / (H, W, n, 4)), so a view taken before a frame loop
    reflects later frames (tests/test_acceptance.py:130-139 relies on that).
    """

    def __init__(self, engine):
        self._eng = engine

    def _shapes(self):
        return self._eng._shapes()

    def __getitem__(self, key):
        shapes = self._shapes()
        if key not in shapes:
            raise KeyError(key)
        return self._eng._read_field(key)

    def __iter__(self):
        return iter(self._shapes())

    def __len__(self):
        return len(self._shapes())


class SegmentationEngine:
    """Per-sequence segmentation state machine on one B200 (engine.py:53-143)."""

    def __init__(self, config, width: int, height: int, device: int | None = None, *,
                 _band=None):
        validate_config(config)
        if width <= 0 or height <= 0:
            raise DimensionError("frame dimensions must be positive")
        self.config = config
        self.width = int(width)
        self.height = int(height)
        self.use_depth = config.mode == "rgbd"
        self.device = default_device() if device is None else int(device)
        self._band = _band
        self.rows = self.height if _band is None else _band[1] - _band[0]
        params = config.gmm if config.algorithm == "gmm" else config.pbas
        self._params = params
        self.gmm_state_dtype = getattr(config, "gmm_state_dtype", "float64")
        gmm_flags = _native.GMM_STATE_F32 if self.gmm_state_dtype == "float32" else 0
        self._h = _Handle(config.algorithm, self.width, self.height, params, self.use_depth,
                          config.seed, self.device, band=_band, gmm_flags=gmm_flags)
        self._gmm_frame_idx = 0
        self.gradient = getattr(config, "pbas_gradient", None) if config.algorithm == "pbas" else None
        if self.gradient is not None:  # opt-in extension, K2G (csrc/pbas.cu)
            if _band is not None:
                self.close()
                raise ConfigError("the PBAS gradient feature needs the whole frame (no row bands)")
            rc = self._h.fn("set_gradient")(self._h.ptr, 1, float(self.gradient.alpha),
                                            float(self.gradient.mean_init))
            _native.check(rc, "set_gradient")

    # ----------------------------------------------------------- surface --
    @property
    def frame_idx(self) -> int:
        if self.config.algorithm == "pbas":
            return int(self._h.fn("get_frame_idx")(self._h.ptr))
        return self._gmm_frame_idx

    @frame_idx.setter
    def frame_idx(self, value: int) -> None:
        if self.config.algorithm == "pbas":
            _native.check(self._h.fn("set_frame_idx")(self._h.ptr, int(value)), "set_frame_idx")
        else:
            self._gmm_frame_idx = int(value)

    @property
    def handle(self) -> int:
        """The raw C-ABI handle (for step_batch users)."""
        return self._h.ptr.value

    @property
    def stream(self) -> int:
        return int(self._h.fn("stream")(self._h.ptr) or 0)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            self._h.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def state_arrays(self) -> StateView:
        return StateView(self)

    def _check_shape(self, shape) -> None:
        if tuple(shape) != (self.rows, self.width, 4):
            raise DimensionError(
                f"frame shape {tuple(shape)} does not match engine "
                f"({self.rows}, {self.width}, 4)"
            )

    def process_frame(self, frame, labels=None):
        """Segment one packed (H, W, 4) uint8 frame; returns the 0/255 mask.

        labels: optional ground truth for this frame ((H, W) uint8, 0 bg /
        1 fg / 2 ignore, frames.py:27-29, or a GroundTruthMask): the kernel
        counts TP/TN/FP/FN as it writes the mask (metrics.compare_masks fused
        into K1/K2), pooled on the device -- read with confusion_counts()."""
        self._check_shape(frame.shape)
        if labels is not None:
            return self._process_eval(frame, labels)
        if _is_torch(frame) and frame.is_cuda:
            return self._process_device(frame)
        if _is_torch(frame):
            frame = frame.numpy()
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        mask = np.empty((self.rows, self.width), dtype=np.uint8)
        rc = self._h.fn("process_host")(self._h.ptr, frame.ctypes.data, mask.ctypes.data, 1)
        _native.check(rc, "process_frame")
        self._gmm_frame_idx += 1
        return mask

    def pack(self, rgb, depth16=None):
        """frames.pack_frame (+ resample_depth when the depth size differs,
        frames.py:46-88) on this engine's device: a CUDA (H, W, 4) frame."""
        from .frames import pack_frame

        return pack_frame(rgb, depth16, device=self.device)

    def apply(self, rgb, depth16=None):
        """apply(rgb, depth) -> mask (the north_star's segmenter call): packs
        RGB + 16-bit depth on the device (frames.py:46-88; depth resampled
        to the RGB size when needed, None = no depth) and segments the frame.
        Returns a CUDA (H, W) uint8 mask tensor."""
        from .frames import pack_frame

        frame = pack_frame(rgb, depth16, device=self.device)
        return self.process_frame(frame)

    def submit(self, frame: np.ndarray, mask_out: np.ndarray) -> None:
        """Asynchronous host path: enqueue H2D + step + D2H into `mask_out`
        and return.  Both buffers must stay alive (and should be pinned) until
        `synchronize()`.  Lets several engines overlap copies and kernels."""
        self._check_shape(frame.shape)
        if mask_out.shape != (self.rows, self.width) or mask_out.dtype != np.uint8:
            raise DimensionError("mask_out must be (H, W) uint8")
        if not (frame.flags["C_CONTIGUOUS"] and frame.dtype == np.uint8
                and mask_out.flags["C_CONTIGUOUS"]):
            raise DimensionError("submit() needs C-contiguous uint8 buffers")
        rc = self._h.fn("process_host")(self._h.ptr, frame.ctypes.data, mask_out.ctypes.data, 0)
        _native.check(rc, "submit")
        self._gmm_frame_idx += 1

    def synchronize(self) -> None:
        _native.check(self._h.fn("sync")(self._h.ptr), "synchronize")

    def _process_device(self, frame):
        import torch

        if frame.dtype != torch.uint8:
            frame = frame.to(torch.uint8)
        if frame.device.index != self.device:
            raise DeviceError(f"frame is on {frame.device}, engine on cuda:{self.device}")
        frame = frame.contiguous()
        mask = torch.empty((self.rows, self.width), dtype=torch.uint8, device=frame.device)
        stream = torch_stream_handle(frame.device)
        self.step_device(frame.data_ptr(), mask.data_ptr(), stream)
        return mask

    def _process_eval(self, frame, labels):
        import torch

        from .metrics import _labels_of

        host = not (_is_torch(frame) and frame.is_cuda)
        dev = torch.device("cuda", self.device)
        lab = _labels_of(labels)
        lab = lab if _is_torch(lab) else torch.from_numpy(np.ascontiguousarray(lab, dtype=np.uint8))
        if tuple(lab.shape) != (self.rows, self.width):
            raise DimensionError(f"mask dimensions {(self.rows, self.width)} do not match ground "
                                 f"truth {tuple(lab.shape)}")  # metrics.py:57-60
        lab = lab.to(device=dev, dtype=torch.uint8).contiguous()
        fr = frame if not host else torch.from_numpy(
            np.ascontiguousarray(frame.numpy() if _is_torch(frame) else frame, dtype=np.uint8))
        fr = fr.to(dev)
        _native.check(self._h.fn("set_eval")(self._h.ptr, ctypes.c_void_p(lab.data_ptr())),
                      "set_eval")
        try:
            mask = self._process_device(fr)
        finally:
            self._h.fn("set_eval")(self._h.ptr, None)
        self._eval_keep = lab  # alive until the stream has consumed it
        return mask.cpu().numpy() if host else mask

    def confusion_counts_device(self, out=None, reset: bool = False):
        """The pooled (tp, tn, fp, fn) of every frame processed with labels
        since the last reset, as a CUDA int64[4] tensor written on the current
        stream (no host sync; feed it to metrics.all_reduce_counts)."""
        import torch

        if out is None:
            out = torch.empty(4, dtype=torch.int64, device=torch.device("cuda", self.device))
        rc = self._h.fn("eval_counts")(self._h.ptr, ctypes.c_void_p(out.data_ptr()), 0, int(reset),
                                       ctypes.c_void_p(torch_stream_handle(out.device)))
        _native.check(rc, "eval_counts")
        return out

    def confusion_counts(self, reset: bool = False):
        """Pooled ConfusionCounts of the frames processed with labels
        (metrics.aggregate_sequence's pooling, metrics.py:94-101)."""
        from .metrics import ConfusionCounts

        return ConfusionCounts.from_sequence(self.confusion_counts_device(reset=reset).tolist())

    def step_device(self, frame_ptr: int, mask_ptr: int, stream: int = 0) -> None:
        """Raw device-pointer step (frame/mask already in HBM)."""
        rc = self._h.fn("step")(self._h.ptr, ctypes.c_void_p(frame_ptr), ctypes.c_void_p(mask_ptr),
                                ctypes.c_void_p(stream))
        _native.check(rc, "step")
        self._gmm_frame_idx += 1

    # ------------------------------------------------------------- state --
    def _shapes(self):
        if self.config.algorithm == "gmm":
            return _GMM_SHAPES
        return {**_PBAS_SHAPES, **_PBAS_GRAD_SHAPES} if self.gradient is not None else _PBAS_SHAPES

    def _field_spec(self, key):
        shapes = self._shapes()
        if key not in shapes:
            raise KeyError(key)
        fields = _native.GMM_FIELDS if self.config.algorithm == "gmm" else _native.PBAS_FIELDS
        shape, dtype = shapes[key](self.rows, self.width, self._params)
        return fields[key], shape, dtype

    def _read_field(self, key) -> np.ndarray:
        fid, shape, dtype = self._field_spec(key)
        self._sync_external()
        out = np.empty(shape, dtype=dtype)
        rc = self._h.fn("read_state")(self._h.ptr, fid, out.ctypes.data, out.nbytes)
        _native.check(rc, f"read_state({key})")
        return out

    def load_state(self, arrays: Mapping) -> None:
        """Write fields given in the reference layout (checkpoint/resume and
        mid-sequence parity seeding)."""
        self._sync_external()
        for key, value in arrays.items():
            fid, shape, dtype = self._field_spec(key)
            arr = np.asarray(value, dtype=dtype, order="C")  # keeps 0-d fields 0-d
            if arr.shape != shape:
                raise DimensionError(f"state field {key}: expected {shape}, got {arr.shape}")
            rc = self._h.fn("write_state")(self._h.ptr, fid, arr.ctypes.data, arr.nbytes)
            _native.check(rc, f"write_state({key})")

    def _sync_external(self) -> None:
        # Steps enqueued on torch's stream (CUDA-tensor inputs) must land
        # before the handle's stream reads or writes the state.
        import sys

        torch = sys.modules.get("torch")
        if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize(self.device)


class MultiStreamEngine:
    """N independent camera streams with the same config and frame size,
    advanced by ONE batched launch per frame (grid over stream x pixel).

    The reference has no multi-stream scheduler; each
    stream here is a full SegmentationEngine (own state, frame_idx and seed:
    `seeds[i]`, default config.seed + i) so `engines[i]` keeps the drop-in
    surface for inspection.
    """

    def __init__(self, config, width: int, height: int, n_streams: int,
                 device: int | None = None, seeds=None):
        import copy

        self.config = config
        self.width, self.height, self.n = int(width), int(height), int(n_streams)
        self.device = default_device() if device is None else int(device)
        seeds = seeds if seeds is not None else [config.seed + i for i in range(self.n)]
        self.engines = []
        for i in range(self.n):
            cfg = copy.copy(config)
            cfg.seed = int(seeds[i])
            self.engines.append(SegmentationEngine(cfg, width, height, self.device))
        self._hs = (ctypes.c_void_p * self.n)(*[e._h.ptr.value for e in self.engines])
        self._fr = (ctypes.c_void_p * self.n)()
        self._mk = (ctypes.c_void_p * self.n)()
        self._fn = (_native.lib().rgbdseg_gmm_step_batch if config.algorithm == "gmm"
                    else _native.lib().rgbdseg_pbas_step_batch)

    def step_ptrs(self, frame_ptrs, mask_ptrs, stream: int = 0, label_ptrs=None) -> None:
        """One batched frame; label_ptrs (device pointers of per-stream
        ground-truth planes, or None) turns on the fused confusion counts."""
        for i in range(self.n):
            self._fr[i] = frame_ptrs[i]
            self._mk[i] = mask_ptrs[i]
        if label_ptrs is not None:
            for e, lp in zip(self.engines, label_ptrs):
                _native.check(e._h.fn("set_eval")(e._h.ptr, ctypes.c_void_p(lp)), "set_eval")
        try:
            rc = self._fn(self._hs, self.n, self._fr, self._mk, ctypes.c_void_p(stream))
        finally:
            if label_ptrs is not None:
                for e in self.engines:
                    e._h.fn("set_eval")(e._h.ptr, None)
        _native.check(rc, "step_batch")
        for e in self.engines:
            e._gmm_frame_idx += 1

    def process(self, frames):
        """frames: torch CUDA uint8 (N, H, W, 4) -> masks (N, H, W)."""
        import torch

        if tuple(frames.shape) != (self.n, self.height, self.width, 4):
            raise DimensionError(f"frames must be ({self.n}, {self.height}, {self.width}, 4)")
        frames = frames.contiguous()
        masks = torch.empty((self.n, self.height, self.width), dtype=torch.uint8,
                            device=frames.device)
        fb, mb = frames.data_ptr(), masks.data_ptr()
        fs, ms = self.height * self.width * 4, self.height * self.width
        self.step_ptrs([fb + i * fs for i in range(self.n)], [mb + i * ms for i in range(self.n)],
                       torch_stream_handle(frames.device))
        return masks

    def close(self):
        for e in self.engines:
            e.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
