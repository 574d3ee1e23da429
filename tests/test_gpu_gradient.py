"""Opt-in PBAS gradient feature on the GPU (K2G pbas_grad_classify_kernel +
pbas_apply_kernel<Code, true>, csrc/pbas.cu) against its CPU checker
oracle_pbas_frame_g (itself pinned in tests/test_pbas_gradient.py): masks,
every state array (incl. the per-sample magnitudes and the previous-frame
sum) bit for bit, on ragged tiles, both intent-code widths, both modes, the
batched multi-stream launch, checkpoint/resume, fused confusion counts and
1080p; alpha = 0 must reproduce the reference algorithm exactly."""

import ctypes

import numpy as np
import pytest

from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import PbasGradient, PbasParams, PipelineConfig

pytestmark = pytest.mark.gpu


def _cfg(n=6, mm=2, mode="rgbd", seed=5, grad=PbasGradient()):
    return PipelineConfig(algorithm="pbas", mode=mode, pbas=PbasParams(n=n, min_matches=mm),
                          seed=seed, pbas_gradient=grad)


def _engine(cfg, w, h):
    from paper_2002_00250_b200.engine import SegmentationEngine

    return SegmentationEngine(cfg, w, h, device=0)


def _compare_run(oracle_mod, cfg, w, h, frames, workers=2):
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=workers)
    with _engine(cfg, w, h) as eng:
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {t}")
        got = {k: v.copy() for k, v in eng.state_arrays().items()}
    want = ref.state_arrays()
    assert set(got) == set(want)
    for k in want:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    return got


@pytest.mark.parametrize("w,h,n,mm,mode,alpha", [
    (45, 31, 6, 2, "rgbd", 10.0),      # ragged in x and y
    (64, 16, 20, 2, "rgbd", 10.0),     # the paper's n, whole tiles
    (45, 13, 20, 1, "rgbd", 10.0),     # n = 20 order statistics, min_matches 1
    (40, 12, 20, 3, "rgbd", 10.0),     # n = 20 with counters
    (64, 16, 20, 2, "rgb_only", 60.0), # large weight
    (33, 9, 40, 2, "rgbd", 4.0),       # u16 intent codes
    (50, 23, 7, 1, "rgb_only", 10.0),
    (37, 19, 9, 3, "rgbd", 25.0),
    (1, 1, 3, 1, "rgbd", 10.0),
    (1, 40, 4, 2, "rgbd", 10.0),
    (70, 1, 4, 2, "rgbd", 10.0),
])
def test_gradient_matches_oracle(oracle_mod, w, h, n, mm, mode, alpha):
    cfg = _cfg(n, mm, mode, seed=w * 7 + h, grad=PbasGradient(alpha=alpha, mean_init=12.0))
    st = _compare_run(oracle_mod, cfg, w, h, synth.sequence("T", w, h, seed=w + h, frames=n + 30))
    assert st["samples_grad"].shape == (h, w, n)


def test_gradient_alpha_zero_is_the_reference_algorithm(oracle_mod):
    w, h, n = 96, 40, 20
    frames = synth.sequence("T", w, h, seed=4, frames=n + 25)
    with _engine(_cfg(n, grad=PbasGradient(alpha=0.0)), w, h) as g, \
            _engine(_cfg(n, grad=None), w, h) as plain:
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(g.process_frame(f), plain.process_frame(f),
                                          err_msg=f"frame {t}")
        pst = plain.state_arrays()
        gst = g.state_arrays()
        for k in pst:
            np.testing.assert_array_equal(gst[k], pst[k], err_msg=k)


def test_gradient_batched_streams_match_oracle(oracle_mod):
    import torch

    from paper_2002_00250_b200.engine import MultiStreamEngine

    w, h, n, ns = 48, 20, 6, 3
    cfg = _cfg(n, seed=100)
    seqs = [synth.sequence("T", w, h, seed=10 + i, frames=n + 20) for i in range(ns)]
    refs = []
    for i in range(ns):
        c = _cfg(n, seed=100 + i)
        refs.append(oracle_mod.OracleEngine(c, w, h, workers=1))
    with MultiStreamEngine(cfg, w, h, ns, device=0) as ms:
        for t in range(n + 20):
            frames = torch.from_numpy(np.stack([s[t] for s in seqs])).cuda()
            masks = ms.process(frames).cpu().numpy()
            for i in range(ns):
                np.testing.assert_array_equal(masks[i], refs[i].process_frame(seqs[i][t]),
                                              err_msg=f"stream {i} frame {t}")
        for i, e in enumerate(ms.engines):
            for k, v in refs[i].state_arrays().items():
                np.testing.assert_array_equal(e.state_arrays()[k], v, err_msg=f"stream {i} {k}")


def test_gradient_checkpoint_resume(oracle_mod):
    w, h, n = 40, 24, 6
    cfg = _cfg(n, seed=9)
    frames = synth.sequence("T", w, h, seed=6, frames=n + 30)
    cut = n + 12
    with _engine(cfg, w, h) as a:
        for f in frames[:cut]:
            a.process_frame(f)
        snap = {k: v.copy() for k, v in a.state_arrays().items()}
        fidx = a.frame_idx
        rest_a = [a.process_frame(f) for f in frames[cut:]]
        final_a = {k: v.copy() for k, v in a.state_arrays().items()}
    with _engine(cfg, w, h) as b:
        b.load_state(snap)
        b.frame_idx = fidx
        assert int(b.state_arrays()["grad_prev_sum"]) == int(snap["grad_prev_sum"])
        rest_b = [b.process_frame(f) for f in frames[cut:]]
        np.testing.assert_array_equal(np.stack(rest_b), np.stack(rest_a))
        for k, v in final_a.items():
            np.testing.assert_array_equal(b.state_arrays()[k], v, err_msg=k)


def test_gradient_fused_confusion_counts(oracle_mod):
    w, h, n = 64, 32, 6
    cfg = _cfg(n, seed=3)
    frames = synth.sequence("T", w, h, seed=8, frames=n + 10)
    rng = np.random.default_rng(1)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    want = np.zeros(4, np.int64)
    with _engine(cfg, w, h) as eng:
        for f in frames:
            lab = rng.integers(0, 3, size=(h, w), dtype=np.uint8)
            got_mask = eng.process_frame(f, labels=lab)
            m = ref.process_frame(f)
            np.testing.assert_array_equal(got_mask, m)
            want += np.array(oracle_mod.compare_masks(m, lab))
        c = eng.confusion_counts()
    assert (c.tp, c.tn, c.fp, c.fn) == tuple(int(v) for v in want)


def test_gradient_rejections():
    from paper_2002_00250_b200 import _native
    from paper_2002_00250_b200.engine import SegmentationEngine
    from paper_2002_00250_b200.errors import ConfigError

    w, h = 32, 8
    frames = synth.sequence("T", w, h, seed=1, frames=2)
    with _engine(_cfg(3, grad=None), w, h) as e:
        e.process_frame(frames[0])
        L = _native.lib()
        assert L.rgbdseg_pbas_set_gradient(e._h.ptr, 1, 10.0, 20.0) == 2  # after the first frame
        assert b"before the first frame" in L.rgbdseg_last_error()
    with pytest.raises(ConfigError):
        SegmentationEngine(_cfg(3), w, h, device=0, _band=(0, 4))
    with _engine(_cfg(3), w, h) as e:
        L = _native.lib()
        assert L.rgbdseg_pbas_set_gradient(e._h.ptr, 1, -1.0, 20.0) == 2
        assert L.rgbdseg_pbas_set_gradient(e._h.ptr, 1, 1.0, 0.0) == 2
        import torch

        fr = torch.from_numpy(frames[0]).cuda()
        m = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        rc = L.rgbdseg_pbas_classify_rows(e._h.ptr, ctypes.c_void_p(fr.data_ptr()),
                                          ctypes.c_void_p(m.data_ptr()), 0, 4, None)
        assert rc == 2
        # switching off before the first frame restores the reference algorithm
        assert L.rgbdseg_pbas_set_gradient(e._h.ptr, 0, 0.0, 0.0) == 0


@pytest.mark.slow
def test_gradient_1080p_matches_oracle(oracle_mod):
    w, h, n = 1920, 1080, 20
    cfg = _cfg(n, seed=77, grad=PbasGradient(alpha=10.0))
    _compare_run(oracle_mod, cfg, w, h, synth.sequence("T", w, h, seed=2, frames=n + 10),
                 workers=oracle_mod.cpu_threads())
