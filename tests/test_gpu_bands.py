"""Row-band PBAS (BASELINE config 5, bands.RowBandPbas) on the GPU with the
peer-memory intent-halo exchange (csrc/peer.cu):

  * 2 and 3 ranks over gloo, all on cuda:0: each rank maps its neighbours'
    mailboxes with CUDA IPC (the multi-GPU code path; on one device the
    "peer" stores land in the same HBM) and synchronises with device flags;
  * 2, 3, 4 and 8 bands in ONE process (connect_local), including several
    frames in flight on one stream, and 8 bands of a 1080p frame against one
    band and the CPU reference;
  * a neighbour that never pushes: the bounded wait reports DeviceError
    instead of hanging the GPU.

Every band runs the kernels with global coordinates; the stitched masks and
state must equal a single-engine run and the CPU oracle bit for bit."""

import ctypes
import os
import socket

import numpy as np
import pytest

from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import PbasParams, PipelineConfig

pytestmark = pytest.mark.gpu

W, H, NF = 96, 37, 30


def _cfg():
    return PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=8), seed=123)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, W=W, H=H):
    import torch
    import torch.distributed as dist

    from paper_2002_00250_b200.bands import RowBandPbas

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    band = RowBandPbas(_cfg(), W, H, rank, world, device=0)
    assert band.link is not None
    band.link.set_timeout(60.0)  # ranks time-slice one GPU here
    frames = synth.sequence("T", W, H, seed=8, frames=NF)
    masks = []
    for f in frames:
        fr = torch.from_numpy(f[band.y0:band.y1].copy()).cuda()
        m = torch.empty((band.rows, W), dtype=torch.uint8, device="cuda")
        band.step(fr, m)
        masks.append(m.cpu().numpy())
    band.status()
    state = {k: v for k, v in band.engine.state_arrays().items()}
    got = [None] * world
    dist.all_gather_object(got, (band.y0, band.y1, np.stack(masks), state))
    if rank == 0:
        np.save(out, np.array(got, dtype=object), allow_pickle=True)
    dist.barrier()
    band.close()
    dist.destroy_process_group()


def _reference(oracle_mod, frames, w, h, cfg):
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    return ref, np.stack([ref.process_frame(f) for f in frames])


@pytest.mark.parametrize("world,w,h", [(2, W, H), (3, W, H), (4, 7680, 48)])
def test_row_band_pbas_ranks_ipc_match_single_engine(oracle_mod, tmp_path, world, w, h):
    # (4, 7680, 48): four ranks at the 8K width of BASELINE config 5, so the
    # mailboxes carry production-size halo rows (7680 codes per boundary)
    import torch.multiprocessing as mp

    out = tmp_path / "bands.npy"
    mp.start_processes(_worker, args=(world, _port(), str(out), w, h), nprocs=world,
                       start_method="spawn", join=True)
    parts = np.load(out, allow_pickle=True)
    ref, ref_masks = _reference(oracle_mod, synth.sequence("T", w, h, seed=8, frames=NF), w, h,
                                _cfg())
    for y0, y1, masks, state in parts:
        np.testing.assert_array_equal(masks, ref_masks[:, y0:y1], err_msg=f"rows {y0}:{y1}")
        for k, v in state.items():
            np.testing.assert_array_equal(v, ref.state_arrays()[k][y0:y1], err_msg=f"{k} {y0}:{y1}")


@pytest.mark.parametrize("nbands", [2, 3, 4, 8])
def test_row_bands_local_peer_links_match_oracle(oracle_mod, nbands):
    # All bands in one process on one device, mailboxes connected directly;
    # every band's frame is enqueued on ONE stream in band order, so a band's
    # pull waits on a push enqueued earlier -- and the consumed flags let the
    # next frames proceed without any host synchronisation in between.
    import torch

    from paper_2002_00250_b200.bands import HaloLink, band_bounds, band_step_p2p
    from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle

    w, h, n = 45, 31, 6
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=n), seed=33)
    frames = synth.sequence("T", w, h, seed=21, frames=n + 25)
    ref, ref_masks = _reference(oracle_mod, frames, w, h, cfg)
    bounds = band_bounds(h, nbands)
    engines = [SegmentationEngine(cfg, w, h, device=0, _band=b) for b in bounds]
    links = [HaloLink(e) for e in engines]
    for i, l in enumerate(links):
        l.connect_local(links[i - 1] if i > 0 else None, links[i + 1] if i < nbands - 1 else None)
    st = ctypes.c_void_p(torch_stream_handle())
    dev_frames = [torch.from_numpy(f).cuda() for f in frames]
    masks = torch.empty((len(frames), h, w), dtype=torch.uint8, device="cuda")
    # edge rows + push of EVERY band first, then interior + pull + apply:
    # stream order must never put a pull ahead of the push it waits for
    from paper_2002_00250_b200 import _native

    L = _native.lib()
    for t, fr in enumerate(dev_frames):
        ptrs = [(ctypes.c_void_p(fr[y0:y1].data_ptr()), ctypes.c_void_p(masks[t, y0:y1].data_ptr()))
                for (y0, y1) in bounds]
        if t < n:
            for e, l, (fp, mp) in zip(engines, links, ptrs):
                band_step_p2p(e, l, fp, mp, st)
            continue
        step = t - n + 1
        for e, l, (fp, mp) in zip(engines, links, ptrs):
            rows = e.rows
            _native.check(L.rgbdseg_pbas_classify_rows(e._h.ptr, fp, mp, 0, rows, st))
            l.push(step, st)
        for e, l, (fp, _) in zip(engines, links, ptrs):
            l.pull(step, st)
            _native.check(L.rgbdseg_pbas_apply(e._h.ptr, fp, st))
    for l in links:
        l.status()
    np.testing.assert_array_equal(masks.cpu().numpy(), ref_masks)
    for e, (y0, y1) in zip(engines, bounds):
        for k, v in e.state_arrays().items():
            np.testing.assert_array_equal(v, ref.state_arrays()[k][y0:y1], err_msg=f"{k} {y0}:{y1}")
    for l in links:
        l.close()
    for e in engines:
        e.close()


def test_halo_wait_times_out_instead_of_hanging():
    import torch

    from paper_2002_00250_b200.bands import HaloLink, band_bounds
    from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle
    from paper_2002_00250_b200.errors import DeviceError

    w, h = 40, 20
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=2), seed=1)
    bounds = band_bounds(h, 2)
    engines = [SegmentationEngine(cfg, w, h, device=0, _band=b) for b in bounds]
    links = [HaloLink(e) for e in engines]
    links[0].connect_local(None, links[1])
    links[1].connect_local(links[0], None)
    links[0].set_timeout(0.05)
    st = ctypes.c_void_p(torch_stream_handle())
    # stale codes in the halo row (as a previous frame would leave them)
    from paper_2002_00250_b200 import _native

    hb, rb = ctypes.c_void_p(), ctypes.c_int64()
    _native.check(_native.lib().rgbdseg_pbas_halo_ptrs(engines[0]._h.ptr, None, None, None,
                                                      ctypes.byref(hb), ctypes.byref(rb)))

    class _Raw:  # device bytes as a torch view (CUDA array interface)
        __cuda_array_interface__ = {"shape": (rb.value,), "typestr": "|u1",
                                    "data": (hb.value, False), "version": 3}

    halo = torch.as_tensor(_Raw(), device="cuda")
    halo.fill_(0x03)
    torch.cuda.synchronize()
    links[0].pull(1, st)  # band 1 never pushes step 1
    torch.cuda.synchronize()
    with pytest.raises(DeviceError, match="timed out"):
        links[0].check_error()  # host-mapped flag, no device sync
    assert bool((halo == 0xFF).all()), "a timed-out pull must leave 'no intent' in the halo"
    with pytest.raises(DeviceError, match="timed out"):
        links[0].status()
    torch.cuda.synchronize()
    for l in links:
        l.close()
    for e in engines:
        e.close()


def test_eight_bands_1080p_match_one_band_and_oracle(oracle_mod):
    # a frame split into 8 row bands (the 8-GPU layout, here
    # 8 handles on one device linked through their peer-memory mailboxes)
    # must equal one band and the CPU reference bit for bit, at full HD with
    # the paper's n = 20 (30 frames: 20 warm-up + 10 with neighbour updates).
    import torch

    from paper_2002_00250_b200 import _native
    from paper_2002_00250_b200.bands import HaloLink, band_bounds
    from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle

    w, h, nb = 1920, 1080, 8
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=20), seed=77)
    frames = synth.sequence("T", w, h, seed=2, frames=30)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=oracle_mod.cpu_threads())
    one = SegmentationEngine(cfg, w, h, device=0)
    bounds = band_bounds(h, nb)
    engines = [SegmentationEngine(cfg, w, h, device=0, _band=b) for b in bounds]
    links = [HaloLink(e) for e in engines]
    for i, l in enumerate(links):
        l.connect_local(links[i - 1] if i > 0 else None, links[i + 1] if i < nb - 1 else None)
    L = _native.lib()
    st = ctypes.c_void_p(torch_stream_handle())
    for t, f in enumerate(frames):
        fr = torch.from_numpy(f).cuda()
        mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        ptrs = [(ctypes.c_void_p(fr[y0:y1].data_ptr()), ctypes.c_void_p(mask[y0:y1].data_ptr()))
                for (y0, y1) in bounds]
        step = t - cfg.pbas.n + 1
        for e, l, (fp, mp) in zip(engines, links, ptrs):
            _native.check(L.rgbdseg_pbas_classify_rows(e._h.ptr, fp, mp, 0, e.rows, st))
            if step >= 1:
                l.push(step, st)
        for e, l, (fp, _) in zip(engines, links, ptrs):
            if step >= 1:
                l.pull(step, st)
            _native.check(L.rgbdseg_pbas_apply(e._h.ptr, fp, st))
        want = one.process_frame(fr).cpu().numpy()
        np.testing.assert_array_equal(mask.cpu().numpy(), want, err_msg=f"frame {t}")
        np.testing.assert_array_equal(want, ref.process_frame(f), err_msg=f"frame {t} vs oracle")
    for l in links:
        l.status()
    for k, v in one.state_arrays().items():
        np.testing.assert_array_equal(v, ref.state_arrays()[k], err_msg=k)
        np.testing.assert_array_equal(
            np.concatenate([e.state_arrays()[k] for e in engines]), v, err_msg=f"bands {k}")
    for l in links:
        l.close()
    for e in engines + [one]:
        e.close()
