"""Row-band split of one oversized frame across GPUs (BASELINE config 5).

The reference splits a frame into contiguous row bands for its thread pool
(`np.linspace(0, H, workers + 1)`, pkg/src/rgbdseg/engine.py:48-50) and
applies PBAS neighbour intents sequentially after every band has classified
(engine.py:140-143).  Here each band lives on its own GPU (one process per
GPU, torch.distributed for the plumbing):

  * GMM is purely per-pixel: bands need no exchange at all.
  * PBAS's only cross-pixel effect is the neighbour-update intent
    (pbas.py:479-507): a band's first/last row may ask a pixel of the
    adjacent band to absorb its own value.  Each band therefore ships ONE row
    of intent codes per boundary per direction (W codes: 7.7 KB at 8K) to the
    neighbouring rank, which pulls them from its halo rows in K3.
    Classification reads no neighbour data, so nothing else crosses.
  * The RNG and the in-bounds tests use global (x, y, W, H)
    (rgbdseg_pbas_create_band), so the result is bit-identical to one GPU and
    to the reference for any number of bands.

Per frame, on the current CUDA stream:
  classify edge rows -> copy them out -> NCCL send/recv (overlaps the
  interior classify) -> set halos -> K3 pull-apply.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .engine import SegmentationEngine, torch_stream_handle

NONE_BYTE = 0xFF  # "no intent" (u8 code 0xFF, u16 code 0xFFFF)


def band_bounds(height: int, parts: int):
    """Row bands exactly as the reference engine splits rows (engine.py:48-50)."""
    edges = np.linspace(0, height, parts + 1).astype(np.int64)
    return [(int(edges[i]), int(edges[i + 1])) for i in range(parts)]


def exchange_intent_halos(first_row, last_row, halo_above, halo_below, rank: int, world: int,
                          group=None, wait: bool = True):
    """One-row intent halo exchange between adjacent bands.

    Sends this band's first intent row to rank-1 (it becomes that band's
    halo below) and its last row to rank+1 (their halo above); receives
    rank-1's last row into `halo_above` and rank+1's first row into
    `halo_below`.  At the global top/bottom the halo is "no intent".
    Works with any torch.distributed backend (NCCL on GPUs, gloo on CPU).
    Returns the pending works when wait=False.
    """
    import torch.distributed as dist

    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, first_row, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, halo_above, rank - 1, group))
    else:
        halo_above.fill_(NONE_BYTE)
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, last_row, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, halo_below, rank + 1, group))
    else:
        halo_below.fill_(NONE_BYTE)
    works = dist.batch_isend_irecv(ops) if ops else []
    if wait:
        for w in works:
            w.wait()
        return []
    return works


class RowBandPbas:
    """This rank's band of a frame split across `world` GPUs (PBAS)."""

    def __init__(self, config, width: int, height: int, rank: int, world: int,
                 device: int | None = None, group=None):
        import torch

        self.rank, self.world, self.group = rank, world, group
        self.y0, self.y1 = band_bounds(height, world)[rank]
        self.engine = SegmentationEngine(config, width, height, device, _band=(self.y0, self.y1))
        self.rows = self.y1 - self.y0
        self.width = width
        rb = ctypes.c_int64()
        L = _native.lib()
        _native.check(L.rgbdseg_pbas_halo_ptrs(self.engine._h.ptr, None, None, None, None,
                                               ctypes.byref(rb)), "halo_ptrs")
        dev = torch.device("cuda", self.engine.device)
        self._send = torch.empty((2, rb.value), dtype=torch.uint8, device=dev)
        self._recv = torch.empty((2, rb.value), dtype=torch.uint8, device=dev)
        self._L = L
        self._device_comm = True
        if world > 1:
            import torch.distributed as dist

            self._device_comm = dist.get_backend(group) == "nccl"

    def step(self, band_frame, band_mask) -> None:
        """Segment this band of one frame (device tensors, (rows, W, 4) and
        (rows, W) uint8), exchanging the intent halos with the neighbours."""
        L, h = self._L, self.engine._h.ptr
        st = ctypes.c_void_p(torch_stream_handle(band_frame.device))
        fp, mp = ctypes.c_void_p(band_frame.data_ptr()), ctypes.c_void_p(band_mask.data_ptr())
        n = self.engine.config.pbas.n
        if self.engine.frame_idx < n or self.world == 1:
            # warm-up frames emit no intents; a single band has no neighbour
            _native.check(L.rgbdseg_pbas_classify(h, fp, mp, st), "classify")
            _native.check(L.rgbdseg_pbas_apply(h, fp, st), "apply")
            return
        rows = self.rows
        _native.check(L.rgbdseg_pbas_classify_rows(h, fp, mp, 0, 1, st), "classify edge")
        if rows > 1:
            _native.check(L.rgbdseg_pbas_classify_rows(h, fp, mp, rows - 1, rows, st),
                          "classify edge")
        s0, s1 = self._send[0], self._send[1]
        _native.check(L.rgbdseg_pbas_copy_edges(h, ctypes.c_void_p(s0.data_ptr()),
                                                ctypes.c_void_p(s1.data_ptr()), st), "copy_edges")
        if self._device_comm:
            works = exchange_intent_halos(s0, s1, self._recv[0], self._recv[1], self.rank,
                                          self.world, self.group, wait=False)
        if rows > 2:  # interior rows overlap the exchange
            _native.check(L.rgbdseg_pbas_classify_rows(h, fp, mp, 1, rows - 1, st),
                          "classify interior")
        if self._device_comm:
            for w in works:
                w.wait()
        else:  # host-staged exchange (gloo: tests that run several ranks on one GPU)
            import torch

            torch.cuda.current_stream(band_frame.device).synchronize()
            hs, hr = self._send.cpu(), torch.empty_like(self._send, device="cpu")
            exchange_intent_halos(hs[0], hs[1], hr[0], hr[1], self.rank, self.world, self.group)
            self._recv.copy_(hr)
        above = ctypes.c_void_p(self._recv[0].data_ptr()) if self.rank > 0 else None
        below = ctypes.c_void_p(self._recv[1].data_ptr()) if self.rank < self.world - 1 else None
        _native.check(L.rgbdseg_pbas_set_halos(h, above, below, st), "set_halos")
        _native.check(L.rgbdseg_pbas_apply(h, fp, st), "apply")

    def close(self):
        self.engine.close()
