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
    neighbouring band, which pulls them from its halo rows in K3.
    Classification reads no neighbour data, so nothing else crosses.
  * The RNG and the in-bounds tests use global (x, y, W, H)
    (rgbdseg_pbas_create_band), so the result is bit-identical to one GPU and
    to the reference for any number of bands.

Transport: peer memory.  Every band owns a mailbox in its
HBM (csrc/peer.cu); the neighbours map it with CUDA IPC and a one-CTA kernel
stores the edge rows straight into it over NVLink / NVSwitch, synchronised
by device flags -- no host round trip and no NCCL on the data path (NCCL
only reduces the run's counters at the end, bench.py).  Per frame, all on the
band's CUDA stream:

  classify edge rows -> push (peer stores + ready flag) -> classify interior
  (overlaps the transfer) -> pull (wait flag, copy into the halo rows,
  consumed flag) -> K3 pull-apply.

`transport="nccl"` keeps an NCCL send/recv exchange for comparison.
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


def band_neighbours(height: int, world: int, rank: int):
    """(above, below): the nearest ranks whose bands hold rows, or None at
    the frame edge.  With more bands than rows (engine.py:48-50 gives empty
    bands, tests/test_engine.py:120-127) an empty band is skipped: the row
    right below band r's last row is the first row of the next non-empty
    band."""
    b = band_bounds(height, world)
    above = next((r for r in range(rank - 1, -1, -1) if b[r][1] > b[r][0]), None)
    below = next((r for r in range(rank + 1, world) if b[r][1] > b[r][0]), None)
    return above, below


def exchange_intent_halos(first_row, last_row, halo_above, halo_below, rank: int, world: int,
                          group=None, wait: bool = True, peers=None):
    """One-row intent halo exchange between adjacent bands.

    Sends this band's first intent row to rank-1 (it becomes that band's
    halo below) and its last row to rank+1 (their halo above); receives
    rank-1's last row into `halo_above` and rank+1's first row into
    `halo_below`.  At the global top/bottom the halo is "no intent".
    Works with any torch.distributed backend (NCCL on GPUs, gloo on CPU).
    peers: (above, below) ranks (default rank-1 / rank+1; band_neighbours
    when some bands are empty), None at a frame edge.
    Returns the pending works when wait=False.
    """
    import torch.distributed as dist

    above, below = peers if peers is not None else (rank - 1 if rank > 0 else None,
                                                   rank + 1 if rank < world - 1 else None)
    ops = []
    if above is not None:
        ops.append(dist.P2POp(dist.isend, first_row, above, group))
        ops.append(dist.P2POp(dist.irecv, halo_above, above, group))
    else:
        halo_above.fill_(NONE_BYTE)
    if below is not None:
        ops.append(dist.P2POp(dist.isend, last_row, below, group))
        ops.append(dist.P2POp(dist.irecv, halo_below, below, group))
    else:
        halo_below.fill_(NONE_BYTE)
    works = dist.batch_isend_irecv(ops) if ops else []
    if wait:
        for w in works:
            w.wait()
        return []
    return works


def neighbour_handles(mine: bytes, rank: int, world: int, group=None):
    """All-gather the bands' mailbox handles (any torch.distributed backend)
    and return (above, below): the handles of the nearest bands above and
    below that hold rows (empty bands contribute b""), None at the frame's
    top / bottom edge."""
    import torch.distributed as dist

    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    above = next((handles[r] for r in range(rank - 1, -1, -1) if handles[r]), None)
    below = next((handles[r] for r in range(rank + 1, world) if handles[r]), None)
    return above, below


class HaloLink:
    """This band's peer-memory mailbox (rgbdseg_halo_link_*, csrc/peer.cu)."""

    def __init__(self, engine):
        self._L = _native.lib()
        self.device = engine.device
        self._engine = engine  # keeps the band's intent map alive
        h = ctypes.c_void_p()
        _native.check(self._L.rgbdseg_halo_link_create(engine._h.ptr, self.device, ctypes.byref(h)),
                      "halo_link_create")
        self.ptr = h

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(_native.IPC_HANDLE_BYTES)
        _native.check(self._L.rgbdseg_halo_link_export(self.ptr, buf), "halo_link_export")
        return buf.raw

    def connect(self, above: bytes | None, below: bytes | None) -> None:
        """Map the neighbours' mailboxes (IPC handles from other processes)."""
        a = ctypes.create_string_buffer(above, len(above)) if above else None
        b = ctypes.create_string_buffer(below, len(below)) if below else None
        _native.check(self._L.rgbdseg_halo_link_connect(self.ptr, a, b), "halo_link_connect")

    def connect_local(self, above: "HaloLink | None", below: "HaloLink | None") -> None:
        """Neighbour bands owned by this process (same or peer device)."""
        _native.check(self._L.rgbdseg_halo_link_connect_local(
            self.ptr, above.ptr if above else None, below.ptr if below else None),
            "halo_link_connect_local")

    def push(self, step: int, stream) -> None:
        _native.check(self._L.rgbdseg_halo_link_push(self.ptr, step, stream), "halo_link_push")

    def pull(self, step: int, stream) -> None:
        _native.check(self._L.rgbdseg_halo_link_pull(self.ptr, step, stream), "halo_link_pull")

    def set_timeout(self, seconds: float) -> None:
        _native.check(self._L.rgbdseg_halo_link_set_timeout(self.ptr, int(seconds * 1e9)),
                      "halo_link_set_timeout")

    def status(self) -> None:
        """Synchronise the device and raise DeviceError if a wait timed out."""
        _native.check(self._L.rgbdseg_halo_link_status(self.ptr), "halo exchange")

    def check_error(self) -> None:
        """Raise DeviceError if a wait of an earlier step timed out (reads the
        host-mapped error word: no device sync, so a timeout surfaces at the
        latest on the step after the one that hit it, or at status())."""
        if self._L.rgbdseg_halo_link_error(self.ptr) == 1:
            from .errors import DeviceError

            raise DeviceError("halo exchange: a peer-memory wait timed out; the affected "
                              "frame applied no cross-band neighbour updates")

    def close(self) -> None:
        if self.ptr:
            self._L.rgbdseg_halo_link_destroy(self.ptr)
            self.ptr = None


def band_step_p2p(engine, link, frame, mask, stream) -> None:
    """One frame of one band with the peer-memory halo exchange (frame and
    mask: device pointers of the band's rows; stream: cudaStream_t)."""
    L, h = _native.lib(), engine._h.ptr
    n = engine.config.pbas.n
    fidx = engine.frame_idx
    if fidx < n or link is None:  # warm-up frames emit no intents
        _native.check(L.rgbdseg_pbas_classify(h, frame, mask, stream), "classify")
        _native.check(L.rgbdseg_pbas_apply(h, frame, stream), "apply")
        return
    link.check_error()
    step = fidx - n + 1
    rows = engine.rows
    _native.check(L.rgbdseg_pbas_classify_rows(h, frame, mask, 0, 1, stream), "classify edge")
    if rows > 1:
        _native.check(L.rgbdseg_pbas_classify_rows(h, frame, mask, rows - 1, rows, stream),
                      "classify edge")
    link.push(step, stream)
    if rows > 2:  # interior rows overlap the transfer
        _native.check(L.rgbdseg_pbas_classify_rows(h, frame, mask, 1, rows - 1, stream),
                      "classify interior")
    link.pull(step, stream)
    _native.check(L.rgbdseg_pbas_apply(h, frame, stream), "apply")


class RowBandPbas:
    """This rank's band of a frame split across `world` GPUs (PBAS)."""

    def __init__(self, config, width: int, height: int, rank: int, world: int,
                 device: int | None = None, group=None, transport: str = "p2p"):
        import torch

        if transport not in ("p2p", "nccl"):
            raise ValueError(f"transport must be 'p2p' or 'nccl', not {transport!r}")
        self.rank, self.world, self.group = rank, world, group
        self.transport = transport
        self.y0, self.y1 = band_bounds(height, world)[rank]
        self.rows = self.y1 - self.y0
        self.peers = band_neighbours(height, world, rank)
        # more bands than rows: an empty band has no engine and steps as a
        # no-op; its neighbours link past it (band_neighbours)
        self.engine = (SegmentationEngine(config, width, height, device, _band=(self.y0, self.y1))
                       if self.rows > 0 else None)
        self.width = width
        self._L = _native.lib()
        self.link = None
        if world > 1 and transport == "p2p":
            import torch.distributed as dist

            if self.engine is not None:
                self.link = HaloLink(self.engine)
            mine = self.link.export() if self.link is not None else b""
            above, below = neighbour_handles(mine, rank, world, group)
            if self.link is not None:
                self.link.connect(above, below)
            dist.barrier(group)  # every mailbox mapped before the first push
        elif world > 1 and self.engine is not None:
            import torch.distributed as dist

            if dist.get_backend(group) != "nccl":
                raise ValueError("transport='nccl' needs an NCCL process group")
            rb = ctypes.c_int64()
            _native.check(self._L.rgbdseg_pbas_halo_ptrs(self.engine._h.ptr, None, None, None,
                                                         None, ctypes.byref(rb)), "halo_ptrs")
            dev = torch.device("cuda", self.engine.device)
            self._send = torch.empty((2, rb.value), dtype=torch.uint8, device=dev)
            self._recv = torch.empty((2, rb.value), dtype=torch.uint8, device=dev)

    def step(self, band_frame, band_mask) -> None:
        """Segment this band of one frame (device tensors, (rows, W, 4) and
        (rows, W) uint8), exchanging the intent halos with the neighbours."""
        if self.engine is None:  # empty band (more bands than rows)
            return
        st = ctypes.c_void_p(torch_stream_handle(band_frame.device))
        fp, mp = ctypes.c_void_p(band_frame.data_ptr()), ctypes.c_void_p(band_mask.data_ptr())
        if self.world == 1 or self.transport == "p2p":
            band_step_p2p(self.engine, self.link, fp, mp, st)
            return
        L, h = self._L, self.engine._h.ptr
        if self.engine.frame_idx < self.engine.config.pbas.n:
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
        works = exchange_intent_halos(s0, s1, self._recv[0], self._recv[1], self.rank,
                                      self.world, self.group, wait=False, peers=self.peers)
        if rows > 2:  # interior rows overlap the exchange
            _native.check(L.rgbdseg_pbas_classify_rows(h, fp, mp, 1, rows - 1, st),
                          "classify interior")
        for w in works:
            w.wait()
        above = ctypes.c_void_p(self._recv[0].data_ptr()) if self.peers[0] is not None else None
        below = ctypes.c_void_p(self._recv[1].data_ptr()) if self.peers[1] is not None else None
        _native.check(L.rgbdseg_pbas_set_halos(h, above, below, st), "set_halos")
        _native.check(L.rgbdseg_pbas_apply(h, fp, st), "apply")

    def status(self) -> None:
        """Raise if a peer-memory wait timed out (synchronises the device)."""
        if self.link is not None:
            self.link.status()

    def close(self):
        if self.link is not None:
            self.link.close()
            self.link = None
        if self.engine is not None:
            self.engine.close()
