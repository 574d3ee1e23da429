"""The reference's behavioural acceptance criteria on the device path
(tests/test_acceptance.py:142-197): frames go through apply(rgb, depth16)
(device pack, frames.py:46-88), segmentation, and the device confusion
counts (metrics.compare_masks, metrics.py:50-69)."""

import numpy as np
import pytest

from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig

pytestmark = pytest.mark.gpu


def _run_scene(spec, algorithm, mode, gmm=None):
    from paper_2002_00250_b200.engine import SegmentationEngine

    cfg = PipelineConfig(algorithm=algorithm, mode=mode, gmm=gmm or GmmParams(), pbas=PbasParams())
    out = []
    with SegmentationEngine(cfg, spec.width, spec.height, device=0) as eng:
        for t in range(spec.frames):
            rgb, d16, gt = synth.scene_frame(spec, t)
            out.append((eng.apply(rgb, d16 if mode == "rgbd" else None), gt))
    return out


@pytest.mark.parametrize("algorithm", ["gmm", "pbas"])
@pytest.mark.parametrize("mode", ["rgb_only", "rgbd"])
def test_criterion_4_static_burn_in_is_empty(algorithm, mode):
    # tests/test_acceptance.py:142-152: frames 100-119 of a static scene
    spec = synth.SceneSpec("static", frames=120)
    masks = _run_scene(spec, algorithm, mode)
    assert sum(int(m.count_nonzero()) for m, _ in masks[100:120]) == 0


@pytest.mark.parametrize("algorithm", ["gmm", "pbas"])
def test_criterion_5_colour_camouflage_needs_depth(algorithm):
    # tests/test_acceptance.py:164-181: tau = 4 for GMM in both modes;
    # rgb_only Si < 0.1, rgbd Si > 0.9 over the frames with a GT object.
    from paper_2002_00250_b200.frames import confusion_counts

    spec = synth.SceneSpec("colour_camouflage")
    si = {}
    for mode in ("rgb_only", "rgbd"):
        tp = fp = fn = 0
        for mask, gt in _run_scene(spec, algorithm, mode, gmm=GmmParams(tau=4.0)):
            if not gt.any():
                continue
            c = confusion_counts(mask, (gt > 0).astype(np.uint8))
            tp, fp, fn = tp + c[0], fp + c[2], fn + c[3]
        si[mode] = tp / (tp + fp + fn) if tp + fp + fn else 0.0
    assert si["rgb_only"] < 0.1, si
    assert si["rgbd"] > 0.9, si


# ------------------------------------------- criteria 3 and 7, engine surface
import ctypes  # noqa: E402
import hashlib  # noqa: E402

import golden_util as gu  # noqa: E402
from test_acceptance_golden import criterion3_frames, criterion7_spec  # noqa: E402


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _state_sha(st, keys):
    return [_sha(st[k]) for k in keys]


def test_criterion_3_gmm_invariants_every_frame():
    # tests/test_acceptance.py:125-139 on the device engine: after every one
    # of 500 noisy frames the weights of every pixel sum to 1 within 1e-9 and
    # every variance is >= 1 (read through the live state view); masks, the
    # per-frame extremes and the final state equal the reference's own run
    # (tests/golden/accept_c3.npz).
    from paper_2002_00250_b200.engine import SegmentationEngine

    fx = gu.load("accept_c3.npz")
    with SegmentationEngine(PipelineConfig(algorithm="gmm", mode="rgbd", workers=2), 64, 64,
                            device=0) as eng:
        state = eng.state_arrays()
        for t, frame in enumerate(criterion3_frames()):
            m = eng.process_frame(frame)
            np.testing.assert_array_equal(np.packbits(m > 0), fx["masks"][t], err_msg=f"frame {t}")
            dev = max(float(np.abs(state[k].sum(axis=2) - 1.0).max()) for k in ("rgb_w", "d_w"))
            vmin = min(float(state[k].min()) for k in ("rgb_var", "d_var"))
            assert dev <= 1e-9 and vmin >= 1.0, (t, dev, vmin)
            assert (dev, vmin) == (fx["wsum_dev"][t], fx["var_min"][t]), t
        assert _state_sha(eng.state_arrays(), fx["state_keys"]) == list(fx["state_sha"])


def _c7_frames(eng_pack):
    spec = criterion7_spec()
    return [eng_pack(*synth.scene_frame(spec, t)[:2]) for t in range(spec.frames)]


def _bands_pbas_run(cfg, frames, w, h, nb):
    """PBAS on nb row bands of one device linked through their peer-memory
    mailboxes (csrc/peer.cu), the per-GPU schedule of bands.band_step_p2p
    split in two phases so every push is enqueued before any pull."""
    import torch

    from paper_2002_00250_b200 import _native
    from paper_2002_00250_b200.bands import HaloLink, band_bounds
    from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle

    L = _native.lib()
    st = ctypes.c_void_p(torch_stream_handle())
    bounds = [b for b in band_bounds(h, nb) if b[1] > b[0]]
    engines = [SegmentationEngine(cfg, w, h, device=0, _band=b) for b in bounds]
    links = [HaloLink(e) for e in engines]
    for i, l in enumerate(links):
        l.connect_local(links[i - 1] if i > 0 else None, links[i + 1] if i < len(links) - 1 else None)
    masks = []
    for fr in frames:
        mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        step = engines[0].frame_idx - cfg.pbas.n + 1
        ptrs = [(ctypes.c_void_p(fr[y0:y1].data_ptr()), ctypes.c_void_p(mask[y0:y1].data_ptr()))
                for (y0, y1) in bounds]
        for e, l, (fp, mp) in zip(engines, links, ptrs):
            if step >= 1:
                _native.check(L.rgbdseg_pbas_classify_rows(e._h.ptr, fp, mp, 0, 1, st))
                if e.rows > 1:
                    _native.check(L.rgbdseg_pbas_classify_rows(e._h.ptr, fp, mp, e.rows - 1,
                                                               e.rows, st))
                l.push(step, st)
                if e.rows > 2:
                    _native.check(L.rgbdseg_pbas_classify_rows(e._h.ptr, fp, mp, 1, e.rows - 1, st))
            else:
                _native.check(L.rgbdseg_pbas_classify(e._h.ptr, fp, mp, st))
        for e, l, (fp, _) in zip(engines, links, ptrs):
            if step >= 1:
                l.pull(step, st)
            _native.check(L.rgbdseg_pbas_apply(e._h.ptr, fp, st))
        masks.append(mask.cpu().numpy())
    for l in links:
        l.status()
    parts = [e.state_arrays() for e in engines]
    state = {k: np.concatenate([p[k] for p in parts], axis=0) for k in parts[0]}
    for l in links:
        l.close()
    for e in engines:
        e.close()
    return masks, state


@pytest.mark.parametrize("algorithm", ["gmm", "pbas"])
def test_criterion_7_bit_identical_across_batches_and_bands(algorithm):
    # tests/test_acceptance.py:200-233 (masks and final state identical for
    # 1 / 4 / 8 workers) on the device: the 160x120x200 colour_camouflage
    # scene through (a) one engine, (b) batched launches of 3 and 8 streams
    # carrying the same sequence, (c) 2 and 4 row bands (PBAS: linked by
    # peer-memory intent halos; GMM: independent sub-frames, as the
    # reference's bands) -- every mask and the final state equal the
    # reference engine's run (tests/golden/accept_c7.npz).
    import torch

    from paper_2002_00250_b200.bands import band_bounds
    from paper_2002_00250_b200.engine import MultiStreamEngine, SegmentationEngine

    fx = gu.load("accept_c7.npz")
    w, h = 160, 120
    cfg = PipelineConfig(algorithm=algorithm, mode="rgbd", seed=42)
    gm, keys, sha = fx[f"{algorithm}_masks"], fx[f"{algorithm}_state_keys"], fx[f"{algorithm}_state_sha"]
    with SegmentationEngine(cfg, w, h, device=0) as eng:
        frames = _c7_frames(eng.pack)
        assert [_sha(f.cpu().numpy()) for f in frames] == list(fx["frame_sha"])  # device pack
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(np.packbits(eng.process_frame(f).cpu().numpy() > 0),
                                          gm[t], err_msg=f"1 engine, frame {t}")
        assert _state_sha(eng.state_arrays(), keys) == list(sha)
    for n in (3, 8):
        with MultiStreamEngine(cfg, w, h, n, device=0, seeds=[42] * n) as ms:
            for t, f in enumerate(frames):
                out = ms.process(f.unsqueeze(0).expand(n, h, w, 4).contiguous()).cpu().numpy()
                for s in range(n):
                    np.testing.assert_array_equal(np.packbits(out[s] > 0), gm[t],
                                                  err_msg=f"batch {n} stream {s} frame {t}")
            for s in range(n):
                assert _state_sha(ms.engines[s].state_arrays(), keys) == list(sha), (n, s)
    for nb in (2, 4):
        if algorithm == "pbas":
            masks, state = _bands_pbas_run(cfg, frames, w, h, nb)
        else:
            bounds = band_bounds(h, nb)
            subs = [SegmentationEngine(cfg, w, y1 - y0, device=0) for y0, y1 in bounds]
            masks = []
            for f in frames:
                masks.append(np.concatenate([e.process_frame(f[y0:y1].contiguous()).cpu().numpy()
                                             for e, (y0, y1) in zip(subs, bounds)]))
            parts = [e.state_arrays() for e in subs]
            state = {k: np.concatenate([p[k] for p in parts], axis=0) for k in parts[0]}
            for e in subs:
                e.close()
        for t, m in enumerate(masks):
            np.testing.assert_array_equal(np.packbits(m > 0), gm[t], err_msg=f"{nb} bands, frame {t}")
        assert _state_sha(state, keys) == list(sha), nb


def test_engine_surface_more_workers_and_bands_than_rows(oracle_mod):
    # tests/test_engine.py:120-127: PBAS with workers=8 on a 5x3 frame --
    # empty bands are harmless.  The device engine ignores `workers`; row
    # bands with more bands than rows skip the empty ones (band_neighbours).
    from paper_2002_00250_b200.engine import SegmentationEngine

    cfg = PipelineConfig(algorithm="pbas", workers=8)
    frame = np.full((3, 5, 4), 10, dtype=np.uint8)
    ref = oracle_mod.OracleEngine(cfg, 5, 3, workers=8)
    with SegmentationEngine(cfg, 5, 3, device=0) as eng:
        for t in range(25):
            mask = eng.process_frame(frame)
            np.testing.assert_array_equal(mask, ref.process_frame(frame), err_msg=f"frame {t}")
    assert mask.shape == (3, 5)
    import torch

    frames = [torch.from_numpy(f).cuda() for f in synth.sequence("T", 32, 3, seed=2, frames=40)]
    cfg2 = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=6), seed=3)
    masks, state = _bands_pbas_run(cfg2, frames, 32, 3, 8)  # 8 bands, 3 rows: 5 empty
    ref2 = oracle_mod.OracleEngine(cfg2, 32, 3, workers=1)
    for t, f in enumerate(frames):
        np.testing.assert_array_equal(masks[t], ref2.process_frame(f.cpu().numpy()), err_msg=f"{t}")
    for k, v in ref2.state_arrays().items():
        np.testing.assert_array_equal(state[k], v, err_msg=k)


def test_process_sequence_errors_name_the_frame_index():
    # tests/test_engine.py:65-78: a frame that fails to load / changes size
    # raises SequenceError naming its index.
    from paper_2002_00250_b200.errors import SequenceError
    from paper_2002_00250_b200.sequence import MemorySequence, process_sequence

    rgb = [np.full((12, 16, 3), 40, np.uint8) for _ in range(12)]
    d16 = [np.full((12, 16), 30000, np.uint16) for _ in range(12)]

    class Corrupt(MemorySequence):
        def load(self, i):
            if i == 7:
                raise ValueError("not a png")
            return super().load(i)

    cfg = PipelineConfig(algorithm="gmm", mode="rgbd")
    with pytest.raises(SequenceError, match="frame 7"):
        process_sequence(Corrupt(rgb, d16), cfg, device=0)
    rgb2 = list(rgb)
    rgb2[9] = np.zeros((9, 9, 3), np.uint8)
    with pytest.raises(SequenceError, match="frame 9"):
        process_sequence(MemorySequence(rgb2), PipelineConfig(algorithm="gmm", mode="rgb_only"),
                         device=0)
    with pytest.raises(SequenceError):
        process_sequence(MemorySequence([]), cfg, device=0)
