"""Device-side input staging and evaluation around the hot path.

  pack_frame(rgb, depth16)   frames.scale_depth_map + resample_depth +
                             pack_frame (pkg/src/rgbdseg/frames.py:46-88) as
                             one sm_100a kernel (csrc/frames.cu), bit-exact;
  confusion_counts(mask, gt) metrics.compare_masks (metrics.py:50-69) as a
                             warp-aggregated device reduction.

Inputs may be numpy arrays (uploaded) or torch CUDA tensors (zero copy);
outputs are torch CUDA tensors.  No CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import DimensionError


def _cuda(x, dtype, device):
    import torch

    if isinstance(x, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(x)).to(device=f"cuda:{device}", dtype=dtype)
    if not x.is_cuda:
        x = x.to(f"cuda:{device}")
    return x.to(dtype).contiguous()


def pack_frame(rgb, depth16=None, device: int = 0, stream: int | None = None):
    """(H, W, 3) u8 rgb + (h, w) u16 depth -> packed (H, W, 4) u8 CUDA frame.

    depth16 may have another resolution (nearest-neighbour resample to the
    RGB size, frames.py:73-88); None packs depth 0 (rgb_only)."""
    import torch

    from .engine import torch_stream_handle

    if rgb.ndim != 3 or rgb.shape[2] != 3:
        raise DimensionError(f"rgb raster must be (H, W, 3), got {tuple(rgb.shape)}")
    h, w = int(rgb.shape[0]), int(rgb.shape[1])
    rgb_d = _cuda(rgb, torch.uint8, device)
    dptr, dw, dh = None, 0, 0
    if depth16 is not None:
        if depth16.ndim != 2:
            raise DimensionError(f"depth map must be (H, W), got {tuple(depth16.shape)}")
        if isinstance(depth16, np.ndarray):
            dep = _cuda(np.asarray(depth16, dtype=np.uint16).view(np.int16), torch.int16, device)
        else:  # 16-bit bit pattern on the device, whatever the integer dtype
            dep = depth16.to(f"cuda:{device}")
            if dep.dtype not in (torch.int16, torch.uint16):
                dep = (dep.to(torch.int32) & 0xFFFF).to(torch.int16)
            dep = dep.contiguous()
        dptr, dh, dw = ctypes.c_void_p(dep.data_ptr()), int(dep.shape[0]), int(dep.shape[1])
    out = torch.empty((h, w, 4), dtype=torch.uint8, device=rgb_d.device)
    st = torch_stream_handle(rgb_d.device) if stream is None else stream
    rc = _native.lib().rgbdseg_pack_frame(ctypes.c_void_p(rgb_d.data_ptr()), w, h, dptr, dw, dh,
                                          ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st))
    _native.check(rc, "pack_frame")
    return out


def confusion_counts(mask, labels, device: int = 0):
    """(tp, tn, fp, fn) of a 0/255 mask against GT labels 0 bg / 1 fg / 2 ignore
    (metrics.compare_masks, metrics.py:50-69), reduced on the device."""
    import torch

    from .engine import torch_stream_handle

    m = _cuda(mask, torch.uint8, device)
    lab = _cuda(labels, torch.uint8, device)
    if m.shape != lab.shape:
        raise DimensionError(f"mask dimensions {tuple(m.shape)} do not match ground truth "
                             f"{tuple(lab.shape)}")
    counts = torch.zeros(4, dtype=torch.int64, device=m.device)
    rc = _native.lib().rgbdseg_confusion_accumulate(
        ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(lab.data_ptr()), m.numel(),
        ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(torch_stream_handle(m.device)))
    _native.check(rc, "confusion_accumulate")
    tp, tn, fp, fn = (int(v) for v in counts.cpu())
    return tp, tn, fp, fn


def median3x3(mask, device: int = 0):
    """Opt-in 3x3 median postprocess of a 0/255 mask (north_star; SURVEY.md D4:
    not part of the reference, off unless called): equals
    scipy.ndimage.median_filter(mask, size=3, mode="reflect").  CUDA tensor out."""
    import torch

    from .engine import torch_stream_handle

    m = _cuda(mask, torch.uint8, device)
    if m.ndim != 2:
        raise DimensionError(f"mask must be (H, W), got {tuple(m.shape)}")
    out = torch.empty_like(m)
    rc = _native.lib().rgbdseg_median3x3(ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                         int(m.shape[1]), int(m.shape[0]),
                                         ctypes.c_void_p(torch_stream_handle(m.device)))
    _native.check(rc, "median3x3")
    return out
