"""Multi-rank row-band PBAS (BASELINE config 5, bands.RowBandPbas) on the GPU:
2 and 3 ranks over gloo, all on cuda:0 (NCCL refuses two ranks per GPU, so
the one-row intent halos are staged through host memory here; on a real
multi-GPU box the same code sends them over NCCL).  Every rank runs the band
kernels with global coordinates; the stitched masks and state must equal a
single-engine run and the CPU oracle bit for bit."""

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


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2002_00250_b200.bands import RowBandPbas

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    band = RowBandPbas(_cfg(), W, H, rank, world, device=0)
    frames = synth.sequence("T", W, H, seed=8, frames=NF)
    masks = []
    for f in frames:
        fr = torch.from_numpy(f[band.y0:band.y1].copy()).cuda()
        m = torch.empty((band.rows, W), dtype=torch.uint8, device="cuda")
        band.step(fr, m)
        masks.append(m.cpu().numpy())
    state = {k: v for k, v in band.engine.state_arrays().items()}
    got = [None] * world
    dist.all_gather_object(got, (band.y0, band.y1, np.stack(masks), state))
    if rank == 0:
        np.save(out, np.array(got, dtype=object), allow_pickle=True)
    band.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_band_pbas_ranks_match_single_engine(oracle_mod, tmp_path, world):
    import torch.multiprocessing as mp

    out = tmp_path / "bands.npy"
    mp.start_processes(_worker, args=(world, _port(), str(out)), nprocs=world,
                       start_method="spawn", join=True)
    parts = np.load(out, allow_pickle=True)
    ref = oracle_mod.OracleEngine(_cfg(), W, H, workers=1)
    ref_masks = np.stack([ref.process_frame(f) for f in synth.sequence("T", W, H, seed=8, frames=NF)])
    for y0, y1, masks, state in parts:
        np.testing.assert_array_equal(masks, ref_masks[:, y0:y1], err_msg=f"rows {y0}:{y1}")
        for k, v in state.items():
            np.testing.assert_array_equal(v, ref.state_arrays()[k][y0:y1], err_msg=f"{k} {y0}:{y1}")
