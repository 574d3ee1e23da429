"""Row-band split (BASELINE config 5) host logic on CPU: world_size 2 and 3
over torch.distributed gloo.

Each rank runs the reference algorithm (the oracle restatement of
_pbas_band with GLOBAL coordinates, pbas.py:344-508) on its band only,
encodes its intents as per-emitter codes (dir<<5 | slot -- the K2/K3 wire
format), exchanges ONE halo row per boundary with
`bands.exchange_intent_halos`, pulls the intents aimed at its own pixels
(the K3 protocol, restated in numpy) and finally gathers its rows.  The
stitched result must equal the single-process reference run bit for bit.
"""

import os
import socket

import numpy as np
import pytest

from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.bands import NONE_BYTE, band_bounds
from paper_2002_00250_b200.config import PbasParams, PipelineConfig

NBR = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1))  # pbas.py:34
W, H, NFRAMES = 29, 17, 26


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg():
    return PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=6), seed=97)


def _pull_apply(state, frame, codes_padded, y0, rows, use_depth):
    """K3 semantics: pixel (y0+ly, x) absorbs its own value into every slot a
    neighbour pointed at it.  codes_padded: (rows+2, W+2), border = NONE."""
    val = frame.copy()
    if not use_depth:
        val[:, :, 3] = 0
    for j, (dy, dx) in enumerate(NBR):
        sub = codes_padded[1 - dy: 1 - dy + rows, 1 - dx: 1 - dx + W]
        hit = (sub != NONE_BYTE) & ((sub >> 5) == j)
        ly, lx = np.nonzero(hit)
        slots = (sub[ly, lx] & 31).astype(np.int64)
        state["samples"][y0 + ly, lx, slots] = val[y0 + ly, lx]


def _worker(rank, world, port, out_path, H=H):
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2002_00250_b200.bands import band_neighbours, exchange_intent_halos

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg()
    frames = synth.sequence("T", W, H, seed=4, frames=NFRAMES)
    state = oracle.pbas_state(W, H, cfg.pbas)
    y0, y1 = band_bounds(H, world)[rank]
    rows = y1 - y0
    peers = band_neighbours(H, world, rank)
    masks = []
    crossing = 0
    for f_idx, frame in enumerate(frames):
        if rows == 0:  # more bands than rows: an empty band is harmless (test_engine.py:120-127)
            masks.append(np.zeros((0, W), dtype=np.uint8))
            continue
        mask = np.zeros((H, W), dtype=np.uint8)
        intents, emitters = oracle.pbas_band_emit(cfg, state, frame, f_idx, y0, y1, mask)
        masks.append(mask[y0:y1].copy())
        if f_idx < cfg.pbas.n:
            continue
        crossing += int(np.count_nonzero((intents[:, 0] < y0) | (intents[:, 0] >= y1)))
        codes = np.full((rows, W), NONE_BYTE, dtype=np.uint8)
        for (ty, tx, slot), (ey, ex) in zip(intents, emitters):
            codes[ey - y0, ex] = (NBR.index((int(ty - ey), int(tx - ex))) << 5) | int(slot)
        first, last = torch.from_numpy(codes[0].copy()), torch.from_numpy(codes[-1].copy())
        above = torch.empty(W, dtype=torch.uint8)
        below = torch.empty(W, dtype=torch.uint8)
        exchange_intent_halos(first, last, above, below, rank, world, peers=peers)
        padded = np.full((rows + 2, W + 2), NONE_BYTE, dtype=np.uint8)
        padded[0, 1:-1] = above.numpy()
        padded[1:-1, 1:-1] = codes
        padded[-1, 1:-1] = below.numpy()
        _pull_apply(state, frame, padded, y0, rows, cfg.mode == "rgbd")
    own = {k: v[y0:y1].copy() for k, v in state.items()}
    gathered = [None] * world
    dist.all_gather_object(gathered, (y0, y1, own, np.stack(masks), crossing))
    if rank == 0:
        np.save(out_path, np.array(gathered, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,h", [(2, H), (3, H), (5, 3)])
def test_row_band_halo_exchange_matches_single_process(oracle_mod, tmp_path, world, h):
    # (5, 3): more bands than rows -- two empty bands, their neighbours
    # exchange halos past them (bands.band_neighbours)
    import torch.multiprocessing as mp

    out = tmp_path / "bands.npy"
    mp.start_processes(_worker, args=(world, _free_port(), str(out), h), nprocs=world,
                       start_method="spawn", join=True)
    parts = np.load(out, allow_pickle=True)

    ref = oracle_mod.OracleEngine(_cfg(), W, h, workers=1)
    frames = synth.sequence("T", W, h, seed=4, frames=NFRAMES)
    ref_masks = np.stack([ref.process_frame(f) for f in frames])
    assert sum(int(p[4]) for p in parts) > 0  # intents really crossed band boundaries
    for y0, y1, own, masks, _ in parts:
        np.testing.assert_array_equal(masks, ref_masks[:, y0:y1])
        for k, v in own.items():
            np.testing.assert_array_equal(v, ref.state_arrays()[k][y0:y1], err_msg=f"{k} rows {y0}:{y1}")


def test_band_bounds_match_reference_linspace():
    # engine.py:48-50
    assert band_bounds(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert band_bounds(4320, 8)[-1] == (3780, 4320)
    assert band_bounds(3, 8)[0] == (0, 0)  # more bands than rows: empty bands (test_engine.py:120-127)


def _handles_worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2002_00250_b200.bands import neighbour_handles

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bytes([rank]) * 64  # stands in for a cudaIpcMemHandle_t
    got = neighbour_handles(mine, rank, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, got)
    if rank == 0:
        np.save(out_path, np.array(gathered, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_link_handles_go_to_adjacent_bands(tmp_path, world):
    # bands.RowBandPbas maps rank-1's mailbox as "above" and rank+1's as
    # "below" (the band order of engine.py:48-50); the frame edges get None
    import torch.multiprocessing as mp

    out = tmp_path / "handles.npy"
    mp.start_processes(_handles_worker, args=(world, _free_port(), str(out)), nprocs=world,
                       start_method="spawn", join=True)
    got = np.load(out, allow_pickle=True)
    for r, (above, below) in enumerate(got):
        assert above == (bytes([r - 1]) * 64 if r > 0 else None)
        assert below == (bytes([r + 1]) * 64 if r < world - 1 else None)


def test_band_neighbours_skip_empty_bands():
    from paper_2002_00250_b200.bands import band_neighbours

    # 3 rows over 5 bands: (0,0) (0,1) (1,1) (1,2) (2,3)
    assert [band_neighbours(3, 5, r) for r in range(5)] == [
        (None, 1), (None, 3), (1, 3), (1, 4), (3, None)]
    assert [band_neighbours(10, 3, r) for r in range(3)] == [(None, 1), (0, 2), (1, None)]
