"""Host side of the metrics path (paper_2002_00250_b200/metrics.py): the
derived indicators and pooling restate the reference's metrics.py:76-101 and
carry its known-answer tests (tests/test_metrics.py:107-166 of the
reference); the device counting is covered in tests/test_gpu_parity.py.  The
multi-rank pool reduction runs over gloo on CPU."""

import os
import socket

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_2002_00250_b200.metrics import (ConfusionCounts, aggregate_sequence, all_reduce_counts,
                                           compute_metrics)


def test_frozen_example():  # reference tests/test_metrics.py:107-112
    r = compute_metrics(ConfusionCounts(tp=100, tn=880, fp=10, fn=10))
    assert r.pwc == pytest.approx(2.0, abs=1e-12)
    assert r.fnr == pytest.approx(10 / 110, rel=1e-12)
    assert r.fpr == pytest.approx(10 / 890, rel=1e-12)
    assert r.si == pytest.approx(100 / 120, rel=1e-12)


def test_perfect_mask():  # :114-116
    r = compute_metrics(ConfusionCounts(tp=5, tn=5, fp=0, fn=0))
    assert (r.pwc, r.fnr, r.fpr, r.si) == (0.0, 0.0, 0.0, 1.0)


def test_undefined_denominators():  # :118-127
    r = compute_metrics(ConfusionCounts(tp=0, tn=10, fp=2, fn=0))
    assert r.fnr is None and r.si is not None
    r = compute_metrics(ConfusionCounts(tp=0, tn=10, fp=0, fn=0))
    assert r.fnr is None and r.si is None
    assert r.pwc is not None and r.fpr is not None
    r = compute_metrics(ConfusionCounts())
    assert (r.pwc, r.fnr, r.fpr, r.si) == (None, None, None, None)


@given(tp=st.integers(0, 10**6), tn=st.integers(0, 10**6), fp=st.integers(0, 10**6),
       fn=st.integers(0, 10**6))
def test_ranges(tp, tn, fp, fn):  # :129-137
    r = compute_metrics(ConfusionCounts(tp, tn, fp, fn))
    if r.pwc is not None:
        assert 0.0 <= r.pwc <= 100.0
    for v in (r.fnr, r.fpr, r.si):
        if v is not None:
            assert 0.0 <= v <= 1.0


def test_aggregation():  # :141-166
    c = ConfusionCounts(3, 4, 5, 6)
    assert aggregate_sequence([c]) == compute_metrics(c)
    c2 = ConfusionCounts(10, 20, 3, 4)
    assert aggregate_sequence([c2, c2]).pwc == pytest.approx(compute_metrics(c2).pwc)
    assert aggregate_sequence([c, c2]).counts == c + c2
    with pytest.raises(ValueError):
        aggregate_sequence([])


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reduce_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pool = torch.tensor([rank + 1, 10 * rank, 2, 0], dtype=torch.int64)
    got = all_reduce_counts(pool)
    if rank == 0:
        np.save(out, np.array([got.tp, got.tn, got.fp, got.fn]))
    dist.barrier()
    dist.destroy_process_group()


def test_all_reduce_counts_sums_rank_pools(tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "c.npy"
    mp.start_processes(_reduce_worker, args=(3, _port(), str(out)), nprocs=3, start_method="spawn",
                       join=True)
    assert np.load(out).tolist() == [6, 30, 6, 0]


def test_process_sequence_validates_like_reference():
    # engine.py:158-162: empty sequence and rgbd without depth fail before
    # any device work
    from paper_2002_00250_b200.config import PipelineConfig
    from paper_2002_00250_b200.errors import SequenceError
    from paper_2002_00250_b200.sequence import MemorySequence, RunStats, process_sequence

    with pytest.raises(SequenceError, match="empty"):
        process_sequence(MemorySequence([]), PipelineConfig(algorithm="gmm"))
    rgb = [np.zeros((4, 4, 3), np.uint8)]
    with pytest.raises(SequenceError, match="depth"):
        process_sequence(MemorySequence(rgb), PipelineConfig(algorithm="gmm", mode="rgbd"))
    with pytest.raises(SequenceError, match="length"):
        MemorySequence(rgb, depth16=[])
    with pytest.raises(SequenceError, match="out_dir"):
        process_sequence(MemorySequence(rgb), PipelineConfig(algorithm="gmm", mode="rgb_only",
                                                             emit_masks=True))
    st = RunStats(frames_processed=4, seconds=2.0)
    assert st.fps == 2.0 and st.seconds_per_frame == 0.5
