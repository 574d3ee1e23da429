"""GPU parity: the sm_100a kernels, called through the C-ABI, against the
reference's own outputs (tests/golden, made by the reference) and against the
CPU restatement (oracle/) on the same seeded inputs.

Bar (BASELINE.json north_star):
  - PBAS: masks and full state bit-exact;
  - GMM: full state bit-exact (compared as bit patterns, so -0 != +0), masks
    bit-exact everywhere.  Only `exp` (CUDA libdevice vs host libm, <= 1 ulp)
    may differ in principle, and it feeds the mask score only (gmm.py:311,
    368); no run here has ever shown a differing mask pixel, so any mismatch
    fails (a prefilter regression cannot hide under a tolerance).
"""

import numpy as np
import pytest

import golden_util as gu
from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig

pytestmark = pytest.mark.gpu



def _engine(cfg, w, h):
    from paper_2002_00250_b200.engine import SegmentationEngine

    return SegmentationEngine(cfg, w, h, device=0)


def _run(cfg, frames):
    h, w = frames[0].shape[:2]
    with _engine(cfg, w, h) as eng:
        masks = [eng.process_frame(f) for f in frames]
        st = {k: v.copy() for k, v in eng.state_arrays().items()}
    return np.stack(masks), st


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def _assert_state_equal(got, expected, keys):
    """Bit for bit: float fields as their bit patterns (-0.0 != +0.0)."""
    for k in keys:
        np.testing.assert_array_equal(_bits(got[k]), _bits(expected[k]), err_msg=k)


# ------------------------------------------------ golden (reference) ------
@pytest.mark.parametrize("name", gu.gmm_cases())
def test_gmm_matches_reference_golden(name):
    fx = gu.load(name)
    masks, st = _run(gu.gmm_config(fx, name), list(fx["frames"]))
    np.testing.assert_array_equal(masks, fx["masks"])
    _assert_state_equal(st, fx, gu.GMM_KEYS)


@pytest.mark.parametrize("name", gu.pbas_cases())
def test_pbas_matches_reference_golden(name):
    fx = gu.load(name)
    masks, st = _run(gu.pbas_config(fx, name), list(fx["frames"]))
    np.testing.assert_array_equal(masks, fx["masks"])
    _assert_state_equal(st, fx, gu.PBAS_KEYS)


def test_device_rng_matches_reference_golden():
    from paper_2002_00250_b200.rng import pixel_keys, rng_stream

    fx = gu.load("rng.npz")
    np.testing.assert_array_equal(pixel_keys(fx["keys"]), fx["values"])
    s, x, y, f = (int(v) for v in fx["stream_key"])
    np.testing.assert_array_equal(rng_stream(s, x, y, f, len(fx["stream"])), fx["stream"])


# ------------------------------------------------ oracle, config sizes ----
def _compare_with_oracle(oracle_mod, cfg, frames, keys):
    """Masks every frame and the final state, bit-exact against the oracle."""
    h, w = frames[0].shape[:2]
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=oracle_mod.cpu_threads())
    with _engine(cfg, w, h) as eng:
        for t, f in enumerate(frames):
            m_ref = ref.process_frame(f)
            m_gpu = eng.process_frame(f)
            mism = int(np.count_nonzero(m_gpu != m_ref))
            assert mism == 0, f"frame {t}: {mism} mask pixels differ"
        st = {k: v.copy() for k, v in eng.state_arrays().items()}
    _assert_state_equal(st, ref.state_arrays(), keys)


@pytest.mark.parametrize("k_rgb,regime", [(3, "T"), (7, "T"), (7, "S"), (3, "S")])
def test_gmm_config1_640x480_vs_oracle(oracle_mod, k_rgb, regime):
    # BASELINE config 1: GMM K=3 (and the paper default 7/3), 640x480, 100 frames.
    frames = synth.sequence(regime, 640, 480, seed=0, frames=100, k_rgb=k_rgb)
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=k_rgb, k_d=3))
    _compare_with_oracle(oracle_mod, cfg, frames, gu.GMM_KEYS)


@pytest.mark.parametrize("mode", ["rgbd", "rgb_only"])
def test_pbas_config2_640x480_vs_oracle(oracle_mod, mode):
    # BASELINE config 2: PBAS N=20, 640x480, moving objects + depth holes.
    frames = synth.sequence("T", 640, 480, seed=1, frames=100)
    cfg = PipelineConfig(algorithm="pbas", mode=mode, pbas=PbasParams(n=20), seed=2)
    _compare_with_oracle(oracle_mod, cfg, frames, gu.PBAS_KEYS)


# ------------------------------------------------ edge cases -------------
EDGE_SIZES = [(1, 1), (1, 37), (37, 1), (13, 17), (129, 3)]


@pytest.mark.parametrize("w,h", EDGE_SIZES)
@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_ragged_and_degenerate_sizes(oracle_mod, w, h, algo):
    rng = np.random.default_rng(w * 1000 + h)
    base = rng.integers(0, 256, size=(h, w, 4), dtype=np.uint8)
    frames = []
    for t in range(30):
        f = base.copy()
        f[rng.random((h, w)) < 0.2] = rng.integers(0, 256, size=4, dtype=np.uint8)
        f[:, :, 3][rng.random((h, w)) < 0.1] = 0
        frames.append(f)
    if algo == "gmm":
        cfg = PipelineConfig(algorithm="gmm", gmm=GmmParams(k_rgb=3, k_d=2))
        keys = gu.GMM_KEYS
    else:
        cfg = PipelineConfig(algorithm="pbas", pbas=PbasParams(n=5), seed=11)
        keys = gu.PBAS_KEYS
    _compare_with_oracle(oracle_mod, cfg, frames, keys)


@pytest.mark.parametrize("k_rgb,k_d,mode", [(10, 5, "rgbd"), (16, 1, "rgb_only"), (8, 4, "rgbd"),
                                            (1, 1, "rgbd")])
def test_gmm_component_counts(oracle_mod, k_rgb, k_d, mode):
    # k outside the unrolled set exercises the generic instantiation.
    frames = synth.sequence("S", 48, 40, seed=4, frames=40, k_rgb=min(k_rgb, 7))
    cfg = PipelineConfig(algorithm="gmm", mode=mode,
                         gmm=GmmParams(k_rgb=k_rgb, k_d=k_d, alpha=0.01))
    _compare_with_oracle(oracle_mod, cfg, frames, gu.GMM_KEYS)


@pytest.mark.parametrize("n,mm", [(1, 1), (2, 2), (7, 1), (20, 1), (20, 3), (20, 20), (31, 2),
                                  (32, 3), (64, 2), (255, 4)])
def test_pbas_buffer_sizes(oracle_mod, n, mm):
    # (20, 1/2): pair scan; (20, 3): counters; other n: runtime-n scans
    # n > 31 switches the intent map to 16-bit codes.
    frames = synth.sequence("T", 40, 24, seed=6, frames=n + 25)
    cfg = PipelineConfig(algorithm="pbas", pbas=PbasParams(n=n, min_matches=mm), seed=n)
    _compare_with_oracle(oracle_mod, cfg, frames, gu.PBAS_KEYS)


def test_gmm_small_var_init_non_lazy(oracle_mod):
    # var_init < VAR_FLOOR disables lazy record loading (floor on unseeded slots).
    frames = synth.sequence("T", 40, 24, seed=9, frames=30)
    cfg = PipelineConfig(algorithm="gmm", gmm=GmmParams(k_rgb=4, k_d=2, var_init=0.25, alpha=0.1))
    _compare_with_oracle(oracle_mod, cfg, frames, gu.GMM_KEYS)


# ------------------------------------------------ engine surface ----------
def test_state_view_is_live():
    # tests/test_acceptance.py:130-139 takes state_arrays() once up front.
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd")
    rng = np.random.default_rng(99)
    with _engine(cfg, 64, 64) as eng:
        state = eng.state_arrays()
        assert set(state) == set(gu.GMM_KEYS)
        for _ in range(60):
            frame = rng.integers(0, 256, size=(64, 64, 4), dtype=np.uint8)
            frame[:, :, 3] = rng.integers(1, 256, size=(64, 64))
            eng.process_frame(frame)
            for key in ("rgb_w", "d_w"):
                assert np.abs(state[key].sum(axis=2) - 1.0).max() <= 1e-9
            for key in ("rgb_var", "d_var"):
                assert state[key].min() >= 1.0


def test_pbas_bounds_every_frame():
    # tests/test_pbas.py:249-262 / acceptance criterion 8
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", seed=2)
    rng = np.random.default_rng(6)
    with _engine(cfg, 12, 10) as eng:
        state = eng.state_arrays()
        for _ in range(60):
            eng.process_frame(rng.integers(0, 256, size=(10, 12, 4), dtype=np.uint8))
            assert state["r_rgb"].min() >= 18.0 and state["r_d"].min() >= 18.0
            assert state["t"].min() >= 2.0 and state["t"].max() <= 200.0


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_burn_in_constant_scene_is_background(algo):
    # tests/test_gmm.py:266-272, tests/test_pbas.py:509-519
    frame = np.full((6, 8, 4), 77, dtype=np.uint8)
    with _engine(PipelineConfig(algorithm=algo, mode="rgbd"), 8, 6) as eng:
        masks = [eng.process_frame(frame) for _ in range(40)]
        if algo == "pbas":
            assert (eng.state_arrays()["samples"] == 77).all()
    assert all(int(m.sum()) == 0 for m in masks)


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_all_invalid_depth_equals_rgb_only(algo):
    # tests/test_pbas.py:536-550 / acceptance criterion 6
    rng = np.random.default_rng(51)
    frames = []
    for _ in range(30):
        f = rng.integers(0, 256, size=(9, 13, 4), dtype=np.uint8)
        f[:, :, 3] = 0
        frames.append(f)
    out = {}
    for mode in ("rgbd", "rgb_only"):
        out[mode], _ = _run(PipelineConfig(algorithm=algo, mode=mode, seed=3), frames)
    np.testing.assert_array_equal(out["rgbd"], out["rgb_only"])


def test_frame_shape_checked():
    from paper_2002_00250_b200.errors import DimensionError

    with _engine(PipelineConfig(algorithm="gmm"), 8, 6) as eng:
        with pytest.raises(DimensionError):
            eng.process_frame(np.zeros((6, 9, 4), dtype=np.uint8))


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_batched_streams_equal_single_engines(algo):
    # The race-detection proxy of the reference (worker-count bit-equality,
    # tests/test_gmm.py:250-264) becomes: batched multi-stream launch ==
    # independent single-stream engines, bit for bit.
    import torch

    from paper_2002_00250_b200.engine import MultiStreamEngine

    n, w, h = 3, 33, 20
    seqs = [synth.sequence("T", w, h, seed=s, frames=30) for s in range(n)]
    cfg = PipelineConfig(algorithm=algo, mode="rgbd", seed=40, pbas=PbasParams(n=8))
    ref = []
    for s in range(n):
        c = PipelineConfig(algorithm=algo, mode="rgbd", seed=40 + s, pbas=PbasParams(n=8))
        ref.append(_run(c, seqs[s]))
    with MultiStreamEngine(cfg, w, h, n, device=0) as ms:
        masks = []
        for t in range(30):
            fr = torch.from_numpy(np.stack([seqs[s][t] for s in range(n)])).cuda()
            masks.append(ms.process(fr).cpu().numpy())
        for s in range(n):
            np.testing.assert_array_equal(np.stack([m[s] for m in masks]), ref[s][0])
            st = {k: v for k, v in ms.engines[s].state_arrays().items()}
            _assert_state_equal(st, ref[s][1], list(ref[s][1]))


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_device_tensor_path_equals_host_path(algo):
    import torch

    frames = synth.sequence("T", 50, 30, seed=8, frames=30)
    cfg = PipelineConfig(algorithm=algo, mode="rgbd", seed=5, pbas=PbasParams(n=6))
    host_masks, host_state = _run(cfg, frames)
    with _engine(cfg, 50, 30) as eng:
        dev = [eng.process_frame(torch.from_numpy(f).cuda()).cpu().numpy() for f in frames]
        st = {k: v for k, v in eng.state_arrays().items()}
    np.testing.assert_array_equal(np.stack(dev), host_masks)
    _assert_state_equal(st, host_state, list(host_state))


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_load_state_resume_mid_sequence(oracle_mod, algo):
    # Checkpoint/resume: seed the device from the oracle's state at frame 20
    # and continue; must match the oracle's uninterrupted run.
    frames = synth.sequence("T", 36, 28, seed=12, frames=40)
    cfg = PipelineConfig(algorithm=algo, mode="rgbd", seed=9, pbas=PbasParams(n=10))
    ref = oracle_mod.OracleEngine(cfg, 36, 28, workers=2)
    for f in frames[:20]:
        ref.process_frame(f)
    with _engine(cfg, 36, 28) as eng:
        eng.load_state(ref.state_arrays())
        eng.frame_idx = ref.frame_idx
        for t, f in enumerate(frames[20:]):
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {20 + t}")
        got = {k: v for k, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), list(got))


# ------------------------------------------------ scalar KATs on device ---
def _gmm1(params, rgb_comps, d_comps=(), mode="rgb_only"):
    eng = _engine(PipelineConfig(algorithm="gmm", mode=mode, gmm=params), 1, 1)
    st = {k: v.copy() for k, v in eng.state_arrays().items()}
    for k, (w, mu, v) in enumerate(rgb_comps):
        st["rgb_w"][0, 0, k], st["rgb_mu"][0, 0, k], st["rgb_var"][0, 0, k] = w, mu, v
    for k, (w, mu, v) in enumerate(d_comps):
        st["d_w"][0, 0, k], st["d_mu"][0, 0, k], st["d_var"][0, 0, k] = w, mu, v
    eng.load_state(st)
    return eng


def _px(rgb, d=0):
    return np.array([[[rgb[0], rgb[1], rgb[2], d]]], dtype=np.uint8)


def test_kat_weight_recurrence_on_device():
    # tests/test_gmm.py:143-150
    eng = _gmm1(GmmParams(k_rgb=2, alpha=0.001),
                [(0.5, [0, 0, 0], 100.0), (0.5, [200, 200, 200], 100.0)])
    eng.process_frame(_px((0, 0, 0)))
    w = eng.state_arrays()["rgb_w"][0, 0]
    assert w[0] == pytest.approx(0.5005, abs=1e-12) and w[1] == pytest.approx(0.4995, abs=1e-12)


def test_kat_least_fit_replacement_on_device():
    # tests/test_gmm.py:165-177
    eng = _gmm1(GmmParams(k_rgb=3), [(0.6, [0, 0, 0], 100.0), (0.1, [50, 50, 50], 400.0),
                                     (0.3, [200, 200, 200], 100.0)])
    eng.process_frame(_px((120, 120, 120)))
    st = eng.state_arrays()
    assert st["rgb_mu"][0, 0, 1].tolist() == [120.0, 120.0, 120.0]
    assert st["rgb_var"][0, 0, 1] == 225.0
    assert st["rgb_w"][0, 0, 1] == pytest.approx(0.05 / 0.95, rel=1e-9)


def test_kat_blend_on_device():
    # tests/test_gmm.py:179-186
    eng = _gmm1(GmmParams(k_rgb=1, alpha=0.5), [(1.0, [10, 10, 10], 16.0)])
    eng.process_frame(_px((12, 10, 10)))
    st = eng.state_arrays()
    assert st["rgb_mu"][0, 0, 0].tolist() == [11.0, 10.0, 10.0]
    assert st["rgb_var"][0, 0, 0] == 10.0


def test_kat_first_frame_and_depth_seed_on_device():
    # tests/test_gmm.py:203-219
    with _engine(PipelineConfig(algorithm="gmm", mode="rgbd"), 1, 1) as eng:
        assert eng.process_frame(_px((40, 80, 120), 200))[0, 0] == 0
    with _engine(PipelineConfig(algorithm="gmm", mode="rgbd"), 1, 1) as eng:
        eng.process_frame(_px((1, 2, 3), 0))
        assert eng.state_arrays()["d_w"][0, 0, 0] == 0.0
        eng.process_frame(_px((1, 2, 3), 77))
        assert eng.state_arrays()["d_w"][0, 0, 0] == 1.0
        assert eng.state_arrays()["d_mu"][0, 0, 0, 0] == 77.0


def test_kat_pbas_camouflage_and_self_update_on_device():
    # tests/test_pbas.py:322-330 (depth catches colour camouflage)
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd")
    with _engine(cfg, 1, 1) as eng:
        st = {k: v.copy() for k, v in eng.state_arrays().items()}
        st["samples"][0, 0, :] = (10, 20, 30, 150)
        eng.load_state(st)
        eng.frame_idx = 20
        assert eng.process_frame(_px((10, 20, 30), 90))[0, 0] == 255
        assert eng.state_arrays()["dmin_d"][0, 0, 0] == 60


@pytest.mark.parametrize("w,h,n", [(64, 24, 20), (96, 17, 5), (32, 40, 32), (64, 20, 33)])
def test_pbas_deferred_intents_state_every_frame(oracle_mod, w, h, n):
    # width % 32 == 0 and n <= 32 selects the deferred-intent mode (intents of
    # frame t applied inside frame t+1's K2, flushed before state access);
    # n = 33 takes the K3 path.  Reading the state after EVERY frame checks
    # the flush against the reference semantics (intents applied at the end
    # of each frame, engine.py:140-143).
    frames = synth.sequence("T", w, h, seed=n, frames=n + 30)
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=n), seed=7 + n)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    with _engine(cfg, w, h) as eng:
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {t}")
            if t >= n - 1 and t % 3 == 0:
                np.testing.assert_array_equal(eng.state_arrays()["samples"],
                                              ref.state_arrays()["samples"], err_msg=f"frame {t}")
        got = {k: v for k, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), gu.PBAS_KEYS)


@pytest.mark.parametrize("nbands", [2, 3])
def test_row_bands_on_one_gpu_match_oracle(oracle_mod, nbands):
    # The config-5 split (bands.py) run on ONE device: each band is its own
    # handle with global coordinates; the one-row intent halos move by
    # device copies instead of NCCL.  Stitched masks and state must equal
    # the single-frame reference run bit for bit.
    import ctypes

    import torch

    from paper_2002_00250_b200 import _native
    from paper_2002_00250_b200.bands import band_bounds
    from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle

    w, h, n = 45, 31, 6
    frames = synth.sequence("T", w, h, seed=21, frames=n + 25)
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=n), seed=33)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    bounds = band_bounds(h, nbands)
    engines = [SegmentationEngine(cfg, w, h, device=0, _band=b) for b in bounds]
    L = _native.lib()
    rb = ctypes.c_int64()
    L.rgbdseg_pbas_halo_ptrs(engines[0]._h.ptr, None, None, None, None, ctypes.byref(rb))
    edges = torch.empty((nbands, 2, rb.value), dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch_stream_handle())
    for t, f in enumerate(frames):
        fr = torch.from_numpy(f).cuda()
        mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
        for i, (e, (y0, y1)) in enumerate(zip(engines, bounds)):
            fp = ctypes.c_void_p(fr[y0:y1].data_ptr())
            mp = ctypes.c_void_p(mask[y0:y1].data_ptr())
            _native.check(L.rgbdseg_pbas_classify_rows(e._h.ptr, fp, mp, 0, y1 - y0, st))
            _native.check(L.rgbdseg_pbas_copy_edges(e._h.ptr, ctypes.c_void_p(edges[i, 0].data_ptr()),
                                                    ctypes.c_void_p(edges[i, 1].data_ptr()), st))
        for i, (e, (y0, y1)) in enumerate(zip(engines, bounds)):
            above = ctypes.c_void_p(edges[i - 1, 1].data_ptr()) if i > 0 else None
            below = ctypes.c_void_p(edges[i + 1, 0].data_ptr()) if i < nbands - 1 else None
            _native.check(L.rgbdseg_pbas_set_halos(e._h.ptr, above, below, st))
            _native.check(L.rgbdseg_pbas_apply(e._h.ptr, ctypes.c_void_p(fr[y0:y1].data_ptr()), st))
        np.testing.assert_array_equal(mask.cpu().numpy(), ref.process_frame(f), err_msg=f"frame {t}")
    for e, (y0, y1) in zip(engines, bounds):
        for k, v in e.state_arrays().items():
            np.testing.assert_array_equal(v, ref.state_arrays()[k][y0:y1], err_msg=f"{k} {y0}:{y1}")
        e.close()


# ------------------------------------------------ next rows: staging + eval
@pytest.mark.parametrize("tag", ["all", "up", "odd", "down", "p720_480"])
def test_device_pack_frame_matches_reference(tag):
    # frames.py:46-88 on the device, against frames the reference packed
    from paper_2002_00250_b200.frames import pack_frame

    fx = gu.load("frames.npz")
    got = pack_frame(fx[f"{tag}_rgb"], fx[f"{tag}_d16"]).cpu().numpy()
    np.testing.assert_array_equal(got, fx[f"{tag}_frame"])


def test_apply_rgb_depth_equals_process_frame_on_packed(oracle_mod):
    # apply(rgb, depth16) == process_frame(pack_frame(rgb, resample(depth16)))
    rng = np.random.default_rng(3)
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=3, k_d=3))
    w, h = 64, 40
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    with _engine(cfg, w, h) as eng:
        for t in range(12):
            rgb = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
            d16 = rng.integers(0, 65536, size=(h // 2, w // 2), dtype=np.uint16)
            d16[rng.random(d16.shape) < 0.1] = 0
            got = eng.apply(rgb, d16).cpu().numpy()
            np.testing.assert_array_equal(got, ref.process_frame(oracle_mod.pack_frame(rgb, d16)))


def test_device_confusion_counts_match_compare_masks(oracle_mod):
    from paper_2002_00250_b200.frames import confusion_counts

    rng = np.random.default_rng(2024)
    for shape in ((32, 32), (1080, 1920), (7, 5)):
        mask = np.where(rng.random(shape) < 0.35, 255, 0).astype(np.uint8)
        labels = rng.choice([0, 1, 2], size=shape, p=[0.5, 0.3, 0.2]).astype(np.uint8)
        assert confusion_counts(mask, labels) == oracle_mod.compare_masks(mask, labels)


@pytest.mark.parametrize("shared", [True, False])
def test_multicamera_pipeline_matches_single_engines(shared):
    # pipeline.MultiCameraPipeline (double-buffered H2D / compute / D2H) must
    # produce, frame by frame, exactly what independent engines produce.
    import torch

    from paper_2002_00250_b200.pipeline import MultiCameraPipeline

    n, w, h, nf = 3, 48, 32, 26
    cfgs = {"gmm": PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=3, k_d=3)),
            "pbas": PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=6), seed=5)}
    seqs = {name: [synth.sequence("T" if name == "pbas" or shared else "S", w, h, seed=s,
                                  frames=nf, k_rgb=3) for s in range(n)] for name in cfgs}
    if shared:
        seqs["pbas"] = seqs["gmm"]
    ref = {}
    for name, cfg in cfgs.items():
        ref[name] = []
        for s in range(n):
            c = PipelineConfig(algorithm=cfg.algorithm, mode="rgbd", gmm=cfg.gmm, pbas=cfg.pbas,
                               seed=cfg.seed + s)
            ref[name].append(_run(c, seqs[name][s])[0])
    with MultiCameraPipeline(cfgs, w, h, n, device=0) as pipe:
        outs = []
        for t in range(nf):
            inp = {name: torch.from_numpy(np.stack([seqs[name][s][t] for s in range(n)])).pin_memory()
                   for name in cfgs}
            out = {name: torch.empty((n, h, w), dtype=torch.uint8).pin_memory() for name in cfgs}
            pipe.submit(inp["gmm"] if shared else inp, out)
            outs.append(out)
        pipe.synchronize()
    for name in cfgs:
        for s in range(n):
            got = np.stack([o[name][s].numpy() for o in outs])
            np.testing.assert_array_equal(got, ref[name][s], err_msg=f"{name} stream {s}")


@pytest.mark.parametrize("shape", [(1, 1), (2, 3), (37, 29), (480, 640), (31, 33)])
def test_median3x3_postprocess_matches_scipy(oracle_mod, shape):
    # opt-in north_star postprocess; oracle = scipy.ndimage.median_filter
    from paper_2002_00250_b200.frames import median3x3

    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    mask = np.where(rng.random(shape) < 0.4, 255, 0).astype(np.uint8)
    np.testing.assert_array_equal(median3x3(mask).cpu().numpy(), oracle_mod.median3x3(mask))


# ------------------------------------------------ C-ABI error paths -------
def test_capi_error_paths_map_to_reference_exceptions():
    import ctypes

    import torch

    from paper_2002_00250_b200 import _native
    from paper_2002_00250_b200.engine import MultiStreamEngine, SegmentationEngine
    from paper_2002_00250_b200.errors import ConfigError, DimensionError, RgbdSegError

    L = _native.lib()
    with SegmentationEngine(PipelineConfig(algorithm="gmm"), 8, 6, device=0) as eng:
        buf = np.empty(10, dtype=np.float64)
        with pytest.raises(DimensionError):  # wrong byte count for rgb_w (6*8*7 doubles)
            _native.check(L.rgbdseg_gmm_read_state(eng._h.ptr, 0, buf.ctypes.data, buf.nbytes))
        with pytest.raises(ConfigError):  # unknown field id
            _native.check(L.rgbdseg_gmm_read_state(eng._h.ptr, 99, buf.ctypes.data, buf.nbytes))
        with pytest.raises(DimensionError):
            eng.load_state({"rgb_w": np.zeros((6, 8, 3))})
        with pytest.raises(DimensionError):  # process_frame shape check (engine.py:101-105)
            eng.process_frame(np.zeros((6, 8, 3), dtype=np.uint8))
    with pytest.raises(ConfigError):  # batch of handles with different parameters
        a = SegmentationEngine(PipelineConfig(algorithm="gmm", gmm=GmmParams(k_rgb=3)), 8, 6, device=0)
        b = SegmentationEngine(PipelineConfig(algorithm="gmm", gmm=GmmParams(k_rgb=4)), 8, 6, device=0)
        hs = (ctypes.c_void_p * 2)(a._h.ptr.value, b._h.ptr.value)
        fr = torch.zeros((2, 6, 8, 4), dtype=torch.uint8, device="cuda")
        mk = torch.empty((2, 6, 8), dtype=torch.uint8, device="cuda")
        fp = (ctypes.c_void_p * 2)(fr[0].data_ptr(), fr[1].data_ptr())
        mp = (ctypes.c_void_p * 2)(mk[0].data_ptr(), mk[1].data_ptr())
        _native.check(L.rgbdseg_gmm_step_batch(hs, 2, fp, mp, None))
    assert issubclass(ConfigError, RgbdSegError)
    # close() is idempotent
    eng = SegmentationEngine(PipelineConfig(algorithm="pbas"), 8, 6, device=0)
    eng.close()
    eng.close()
    with pytest.raises(DimensionError):
        MultiStreamEngine(PipelineConfig(algorithm="gmm"), 8, 6, 2, device=0).process(
            torch.zeros((3, 6, 8, 4), dtype=torch.uint8, device="cuda"))


def test_fast_divide_matches_ieee_divide_on_device():
    # K2's fdiv_rn (csrc/pbas.cu) = the div.rn.f64 fast path without its
    # slow-path branch, used only for operands the host proved in range.
    # Bitwise against `/` on the device over the operand families K2 feeds
    # it (pbas.py:432/448 averages, :462/:464 T steps, :468 1/T, :474/:486
    # u/prob) plus log-uniform pairs across the whole accepted range.
    import ctypes

    import torch

    from paper_2002_00250_b200 import _native

    L = _native.lib()
    rng = np.random.default_rng(7)
    m = 4_000_000

    def check(a, b, what):
        ad = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
        bd = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).cuda()
        bad = ctypes.c_int64(-1)
        _native.check(L.rgbdseg_selftest_fdiv(ctypes.c_void_p(ad.data_ptr()),
                                              ctypes.c_void_p(bd.data_ptr()), ad.numel(),
                                              ctypes.byref(bad)))
        assert bad.value == 0, f"{what}: {bad.value} mismatches"

    tot, ln = np.meshgrid(np.arange(65536.0), np.arange(1.0, 256.0))
    check(tot.ravel(), ln.ravel(), "tot/len exhaustive")
    tt = rng.uniform(2.0, 200.0, m)
    check(np.ones(m), tt, "1/T")
    prob = 1.0 / tt
    u = rng.integers(0, 2**53, m).astype(np.float64) * 2.0**-53
    check(u * prob, prob, "u/prob (u < prob)")
    check(u, prob, "u/prob")
    guard = rng.uniform(1.0, 255.0, m)
    num = np.where(rng.random(m) < 0.5, 1.0, -0.05) * 10.0 ** rng.uniform(-3, 3, m)
    check(num, guard, "t_step/guard")
    # GMM renormalisation w / total (gmm.py:339-343; csrc/gmm.cu rcp_rn_f64 +
    # div_by_rcp = this sequence with the reciprocal hoisted): weights in
    # [1e-140, 1] (or 0), totals in [1e-3, 1.1], and the reference's
    # renormalisation of freshly blended weight vectors
    wts = rng.random(m) * 10.0 ** rng.uniform(-140, 0, m)
    wts[rng.random(m) < 0.05] = 0.0
    check(wts, rng.uniform(1e-3, 1.1, m), "w/total")
    k = 7
    wv = rng.dirichlet(np.ones(k), m // k) * (1.0 - 0.001)
    wv[:, 0] += 0.001
    check(wv.ravel(), np.repeat(wv.sum(axis=1), k), "blended weights / their sum")
    a = 10.0 ** rng.uniform(-145, 145, m) * np.where(rng.random(m) < 0.5, 1.0, -1.0)
    b = 10.0 ** rng.uniform(-145, 145, m)
    check(a, b, "log-uniform")


@pytest.mark.parametrize("r", [0.5, 300.0])
def test_pbas_extreme_radius_thresholds(oracle_mod, r):
    # R < 1: only exact matches count (threshold 1); R > 255: every RGB
    # distance and every valid depth counts (threshold 256, pbas.py:392,
    # :413) -- the edges of the order-statistic scans
    frames = synth.sequence("T", 48, 20, seed=3, frames=40)
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", seed=5,
                         pbas=PbasParams(n=20, r_init=r, r_lower=r))
    _compare_with_oracle(oracle_mod, cfg, frames, gu.PBAS_KEYS)


@pytest.mark.parametrize("w,h", [(64, 37), (96, 8), (32, 1), (640, 480)])
def test_pbas_list_handle_row_ranges(oracle_mod, w, h):
    # A single-band (intent-list) handle classified in uneven row ranges
    # (classify_rows) before one apply: intents across a range boundary must
    # land exactly as in the reference's whole-frame pass.
    import ctypes

    import torch

    from paper_2002_00250_b200 import _native
    from paper_2002_00250_b200.engine import SegmentationEngine, torch_stream_handle

    n = 6
    frames = synth.sequence("T", w, h, seed=17, frames=n + 20)
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=n), seed=29)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    cuts = sorted({0, h, min(h, 5), min(h, 13), h // 2})
    L = _native.lib()
    st = ctypes.c_void_p(torch_stream_handle())
    with SegmentationEngine(cfg, w, h, device=0) as eng:
        for t, f in enumerate(frames):
            fr = torch.from_numpy(f).cuda()
            mask = torch.empty((h, w), dtype=torch.uint8, device="cuda")
            fp, mp = ctypes.c_void_p(fr.data_ptr()), ctypes.c_void_p(mask.data_ptr())
            for r0, r1 in zip(cuts[:-1], cuts[1:]):
                _native.check(L.rgbdseg_pbas_classify_rows(eng._h.ptr, fp, mp, r0, r1, st))
            _native.check(L.rgbdseg_pbas_apply(eng._h.ptr, fp, st))
            np.testing.assert_array_equal(mask.cpu().numpy(), ref.process_frame(f), err_msg=f"frame {t}")
        got = {k: v.copy() for k, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), gu.PBAS_KEYS)


def _labels_seq(frames, seed):
    rng = np.random.default_rng(seed)
    return [rng.choice(3, size=f.shape[:2], p=[0.5, 0.35, 0.15]).astype(np.uint8) for f in frames]


def _counts_oracle(mask, labels):  # metrics.compare_masks, metrics.py:50-69
    fg = mask > 127
    return (int(np.count_nonzero(fg & (labels == 1))), int(np.count_nonzero(~fg & (labels == 0))),
            int(np.count_nonzero(fg & (labels == 0))), int(np.count_nonzero(~fg & (labels == 1))))


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_fused_confusion_counts_pool_like_aggregate_sequence(oracle_mod, algo):
    # process_frame(frame, labels) counts TP/TN/FP/FN inside K1/K2; the pool
    # must equal summing compare_masks over the frames (aggregate_sequence),
    # while masks and state stay bit-exact with the unevaluated run.
    from paper_2002_00250_b200.errors import DimensionError
    from paper_2002_00250_b200.metrics import ConfusionCounts, aggregate_sequence, compute_metrics

    w, h = 67, 29  # ragged: partial warps/blocks
    frames = synth.sequence("T", w, h, seed=5, frames=30)
    labels = _labels_seq(frames, 9)
    cfg = (PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=3, k_d=3))
           if algo == "gmm" else PipelineConfig(algorithm="pbas", mode="rgbd",
                                                pbas=PbasParams(n=8), seed=4))
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    want = ConfusionCounts()
    with _engine(cfg, w, h) as eng:
        for t, (f, lab) in enumerate(zip(frames, labels)):
            m = eng.process_frame(f, labels=lab)
            m_ref = ref.process_frame(f)
            np.testing.assert_array_equal(m, m_ref, err_msg=f"frame {t}")
            want = want + ConfusionCounts(*_counts_oracle(m_ref, lab))
            if t == 10:
                assert eng.confusion_counts() == want
        assert eng.confusion_counts(reset=True) == want
        assert aggregate_sequence([want]) == compute_metrics(eng_counts := want)
        assert eng.confusion_counts() == ConfusionCounts()  # pool restarted
        with pytest.raises(DimensionError):
            eng.process_frame(frames[0], labels=labels[0][:, :-1])
        got = {k: v.copy() for k, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), gu.GMM_KEYS if algo == "gmm" else gu.PBAS_KEYS)
    assert eng_counts.total == sum(int(np.count_nonzero(l != 2)) for l in labels)


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_fused_confusion_counts_batched_streams(algo):
    import torch

    from paper_2002_00250_b200.engine import MultiStreamEngine, torch_stream_handle
    from paper_2002_00250_b200.metrics import ConfusionCounts

    w, h, S = 96, 40, 3
    seqs = [synth.sequence("T", w, h, seed=20 + i, frames=12) for i in range(S)]
    labs = [_labels_seq(seq, 30 + i) for i, seq in enumerate(seqs)]
    cfg = (PipelineConfig(algorithm="gmm", mode="rgbd") if algo == "gmm"
           else PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=6), seed=2))
    want = [ConfusionCounts() for _ in range(S)]
    with MultiStreamEngine(cfg, w, h, S, device=0) as ms:
        for t in range(12):
            fr = torch.from_numpy(np.stack([seqs[i][t] for i in range(S)])).cuda()
            lb = torch.from_numpy(np.stack([labs[i][t] for i in range(S)])).cuda()
            masks = torch.empty((S, h, w), dtype=torch.uint8, device="cuda")
            ms.step_ptrs([fr[i].data_ptr() for i in range(S)], [masks[i].data_ptr() for i in range(S)],
                         torch_stream_handle(), label_ptrs=[lb[i].data_ptr() for i in range(S)])
            mh = masks.cpu().numpy()
            for i in range(S):
                want[i] = want[i] + ConfusionCounts(*_counts_oracle(mh[i], labs[i][t]))
        for i in range(S):
            assert ms.engines[i].confusion_counts() == want[i], f"stream {i}"


@pytest.mark.parametrize("algo,mode", [("gmm", "rgbd"), ("pbas", "rgbd"), ("pbas", "rgb_only")])
def test_process_sequence_matches_reference_pipeline(oracle_mod, algo, mode):
    # engine.py:146-214: resample (depth at another size) + pack + segment per
    # frame; masks to on_mask; labels -> pooled metrics (aggregate_sequence)
    from paper_2002_00250_b200.errors import SequenceError
    from paper_2002_00250_b200.metrics import ConfusionCounts, aggregate_sequence
    from paper_2002_00250_b200.sequence import MemorySequence, process_sequence

    w, h, n = 64, 48, 26
    rng = np.random.default_rng(3)
    base = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    rgbs, deps, labs = [], [], []
    for t in range(n):
        img = base.copy()
        img[10:20, (t % 40):(t % 40) + 12] = 200  # a moving block
        rgbs.append(img)
        d = np.full((h // 2, w // 2), 40000, np.uint16)  # half-size depth: resampled
        d[rng.random(d.shape) < 0.05] = 0
        deps.append(d)
        lab = np.zeros((h, w), np.uint8)
        lab[10:20, (t % 40):(t % 40) + 12] = 1
        lab[0, :] = 2
        labs.append(lab)
    src = MemorySequence(rgbs, deps if mode == "rgbd" else None)
    cfg = (PipelineConfig(algorithm="gmm", mode=mode) if algo == "gmm"
           else PipelineConfig(algorithm="pbas", mode=mode, pbas=PbasParams(n=6), seed=11))
    got = []
    stats = process_sequence(src, cfg, on_mask=lambda fid, m: got.append((fid, m.copy())),
                             labels=labs)
    assert stats.frames_processed == n and len(stats.per_frame_seconds) == n
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    want = ConfusionCounts()
    for t in range(n):
        frame = oracle_mod.pack_frame(rgbs[t], oracle_mod.resample_depth(deps[t], w, h)
                                      if mode == "rgbd" else None)
        m = ref.process_frame(frame)
        assert got[t][0] == src.frame_id(t)
        np.testing.assert_array_equal(got[t][1], m, err_msg=f"frame {t}")
        want = want + ConfusionCounts(*_counts_oracle(got[t][1], labs[t]))
    assert stats.report == aggregate_sequence([want])
    bad = MemorySequence(rgbs[:2] + [rgbs[2][:, :-1]], deps[:3] if mode == "rgbd" else None)
    with pytest.raises(SequenceError, match="differ"):
        process_sequence(bad, cfg)


def test_pbas_load_state_rejects_positions_outside_the_ring():
    # pos must stay < n and len <= n (pbas.py:425-431); the reference's ring
    # write would leave its buffer otherwise -- rejected like bad config
    from paper_2002_00250_b200.errors import ConfigError

    cfg = PipelineConfig(algorithm="pbas", pbas=PbasParams(n=5), seed=1)
    with _engine(cfg, 16, 8) as eng:
        for key, bad in (("pos_rgb", 5), ("pos_d", 200), ("len_rgb", 6)):
            st = eng.state_arrays()[key].copy()
            st[3, 4] = bad
            with pytest.raises(ConfigError):
                eng.load_state({key: st})
        ok = eng.state_arrays()["len_d"].copy()
        ok[:] = 5
        eng.load_state({"len_d": ok})


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_pbas_k2_variants_and_auto_switch(oracle_mod, mode):
    # K2 runs as the row kernel, as the warp-strip kernel that applies
    # in-strip neighbour updates itself, or -- small frames, auto / pinned
    # 3 -- fused with K3 in one cooperative launch.  A fast T decay (t_dec)
    # drives the update rate from ~1/18 to 1/2 within the sequence -- every
    # frame bit-exact with the reference in every mode.  (The auto row ->
    # strip crossover of frames too big to fuse: the 1080p test below.)
    from paper_2002_00250_b200 import _native

    w, h, n = 96, 40, 6
    frames = synth.sequence("T", w, h, seed=12, frames=70)
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", seed=5,
                         pbas=PbasParams(n=n, t_dec=1.0, t_lower=2.0))
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    L = _native.lib()
    seen = set()
    with _engine(cfg, w, h) as eng:
        _native.check(L.rgbdseg_pbas_set_k2_mode(eng._h.ptr, mode))
        for t, f in enumerate(frames):
            seen.add(int(L.rgbdseg_pbas_get_k2_mode(eng._h.ptr)))
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {t}")
        got = {k: v.copy() for k, v in eng.state_arrays().items()}
        last = int(L.rgbdseg_pbas_get_k2_mode(eng._h.ptr))
    _assert_state_equal(got, ref.state_arrays(), gu.PBAS_KEYS)
    assert seen - {1} == ({3} if mode in (0, 3) else {mode}) - {1}  # first get: before any step
    assert last == (3 if mode in (0, 3) else mode)


def test_pbas_auto_switch_rows_to_strips_1080p(oracle_mod):
    # A frame too big for the fused cooperative launch (> 8 pixels per
    # resident thread): auto mode runs the row kernel while few pixels emit
    # neighbour updates and switches to strips once many do (T decays fast
    # here); bit-exact with the reference every frame.
    from paper_2002_00250_b200 import _native

    w, h, n = 1920, 1080, 6
    cfg = PipelineConfig(algorithm="pbas", mode="rgbd", seed=8,
                         pbas=PbasParams(n=n, t_dec=1.0, t_lower=2.0))
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=oracle_mod.cpu_threads())
    L = _native.lib()
    modes = []
    with _engine(cfg, w, h) as eng:
        for t in range(40):
            f = synth.make_frame("T", w, h, 13, t)
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {t}")
            modes.append(int(L.rgbdseg_pbas_get_k2_mode(eng._h.ptr)))
        got = {k: v.copy() for k, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), gu.PBAS_KEYS)
    assert modes[n] == 1 and modes[-1] == 2 and 3 not in modes, modes


@pytest.mark.parametrize("n,mm,mode", [(40, 2, "rgbd"), (7, 3, "rgbd"), (20, 1, "rgb_only"),
                                       (20, 2, "rgbd")])
def test_pbas_tile_variant_code_widths_and_scans(oracle_mod, n, mm, mode):
    # the pinned tile K2 with 16-bit codes (n > 31), the counter scan
    # (min_matches > 2), rgb_only, and the paper's n = 20, against the reference
    from paper_2002_00250_b200 import _native

    w, h = 64, 24
    frames = synth.sequence("T", w, h, seed=31, frames=n + 15)
    cfg = PipelineConfig(algorithm="pbas", mode=mode, seed=9,
                         pbas=PbasParams(n=n, min_matches=mm, t_dec=0.5))
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=1)
    with _engine(cfg, w, h) as eng:
        _native.check(_native.lib().rgbdseg_pbas_set_k2_mode(eng._h.ptr, 2))
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {t}")
        got = {k: v.copy() for k, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), gu.PBAS_KEYS)


# ------------------------------------------- FP32 mask prefilter at tau ---
def _host_score(w, mu, var, x, s):
    """The reference score expression (gmm.py:297-311), in Python floats
    (IEEE f64, host libm exp), over the seeded components of one sub-model."""
    import math

    p = 0.0
    for wk, mk, vk in zip(w, mu, var):
        if wk <= 0.0:
            continue
        d2 = 0.0
        for xc, mc in zip(x, mk):
            dd = xc - mc
            d2 += dd * dd
        p += wk * ((s / (2.0 * math.pi * vk)) * math.exp(-(d2 / (2.0 * vk))))
    return p


def _solve_mu(term, v, s, x0):
    """mu with x0 - mu = sqrt(d2) so that (s/(2 pi v)) exp(-d2/(2v)) ~= term."""
    import math

    d2 = -2.0 * v * math.log(term * 2.0 * math.pi * v / s)
    return x0 - math.sqrt(max(d2, 0.0))


@pytest.mark.parametrize("mode,k", [("rgb_only", 1), ("rgb_only", 3), ("rgbd", 2)])
@pytest.mark.parametrize("tau", [1.0, 4.0])
def test_gmm_prefilter_decisions_at_tau_equal_fp64(mode, k, tau):
    # K1 decides p >= tau from an FP32 estimate unless it lies within
    # 2^-10 tau of tau, where it re-evaluates the exact FP64 expression
    # (csrc/gmm.cu sub_scan / sub_exact_score).  States whose
    # exact score sits at tau (1 +- 2^-10 +- {0, 1e-6, 1e-4}), at the band's
    # inside (tau (1 +- {1e-12, 1e-9, 1e-6, 1e-4, 2^-11})) and outside
    # (+- 2^-9, 1e-2, 0.5): every device decision must equal the host FP64
    # decision of the reference expression (gmm.py:311, :366-368).
    rels = []
    for sgn in (-1.0, 1.0):
        for e in (0.0, 1e-6, -1e-6, 1e-4, -1e-4):
            rels.append(sgn * 2.0 ** -10 + e)
        for e in (1e-12, 1e-9, 1e-6, 1e-4, 2.0 ** -11, 2.0 ** -9, 1e-2, 0.5):
            rels.append(sgn * e)
    s, x0 = 1e4, 100.0
    rng = np.random.default_rng(k * 10 + int(tau))
    cfg = PipelineConfig(algorithm="gmm", mode=mode, gmm=GmmParams(k_rgb=k, k_d=1, tau=tau, s=s))
    npx = len(rels)
    eng = _engine(cfg, npx, 1)
    st = {key: v.copy() for key, v in eng.state_arrays().items()}
    frame = np.zeros((1, npx, 4), np.uint8)
    frame[0, :, :3] = int(x0)
    want = np.empty(npx, np.uint8)
    for i, rel in enumerate(rels):
        target = tau * (1.0 + rel)
        pd = 1.0
        if mode == "rgbd":  # depth sub-model: one component, factor ~0.8-1.2
            dv = float(rng.uniform(200.0, 400.0))
            pdt = float(rng.uniform(0.8, 1.2)) * s / (2.0 * np.pi * dv) / 2.0
            dmu = _solve_mu(pdt, dv, s, 90.0)
            st["d_w"][0, i, 0], st["d_mu"][0, i, 0, 0], st["d_var"][0, i, 0] = 1.0, dmu, dv
            frame[0, i, 3] = 90
            pd = _host_score([1.0], [[dmu]], [dv], [90.0], s)
        ws = rng.dirichlet(np.ones(k)) if k > 1 else np.ones(1)
        term = target / pd  # every component's term: sum_j ws[j] * term = target / pd
        vs = rng.uniform(0.3, 0.7, k) * s / (2.0 * np.pi * term)  # exp factor in (0.3, 0.7)
        mus = np.zeros((k, 3))
        for j in range(k):
            mus[j] = [_solve_mu(term, vs[j], s, x0), x0, x0]
        st["rgb_w"][0, i, :] = ws
        st["rgb_mu"][0, i, :, :] = mus
        st["rgb_var"][0, i, :] = vs
        p = _host_score(ws, mus, vs, [x0] * 3, s) * (pd if mode == "rgbd" else 1.0)
        want[i] = 0 if p >= tau else 255
        # the construction must put p where intended (within 1e-11 relative)
        assert abs(p / target - 1.0) < 1e-11 or abs(rel) >= 1e-2, (rel, p / target - 1.0)
    eng.load_state(st)
    got = eng.process_frame(frame)[0]
    eng.close()
    bad = [(rels[i], int(got[i]), int(want[i])) for i in range(npx) if got[i] != want[i]]
    assert not bad, bad
    # sanity: both decisions occur
    assert (want == 0).any() and (want == 255).any()


def test_gmm_negative_zero_weights_renormalise_like_reference(oracle_mod):
    # -0.0 weights (only in externally loaded state) must stay -0.0 through
    # the renormalisation w / total (gmm.py:339-343): the split divide of the
    # fast path returns +0 for both zeros, so such pixels take the IEEE path.
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=4, k_d=3))
    frames = synth.sequence("T", 24, 16, seed=5, frames=6)
    ref = oracle_mod.OracleEngine(cfg, 24, 16, workers=1)
    for f in frames[:3]:
        ref.process_frame(f)
    st = {key: v.copy() for key, v in ref.state_arrays().items()}
    for key in ("rgb_w", "d_w"):
        z = st[key] == 0.0
        st[key][z] = -0.0
        assert np.signbit(st[key]).any()
    ref.state = {key: v.copy() for key, v in st.items()}
    with _engine(cfg, 24, 16) as eng:
        eng.load_state(st)
        for t, f in enumerate(frames[3:]):
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {3 + t}")
        got = {key: v for key, v in eng.state_arrays().items()}
    assert np.signbit(ref.state_arrays()["rgb_w"]).any()  # -0 survives in the reference
    _assert_state_equal(got, ref.state_arrays(), gu.GMM_KEYS)


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_mixed_input_kinds_stay_ordered(oracle_mod, algo):
    # One engine fed alternately through torch CUDA tensors on a side stream,
    # numpy frames (the handle's own stream), submit() and device pointers on
    # yet another stream: every step must see the previous step's state
    # (the C-ABI orders a step after the handle's last one when the stream
    # changes), so masks and state equal the oracle's sequential run.
    import torch

    w, h, n = 640, 480, 16
    cfg = (PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=7, k_d=3))
           if algo == "gmm" else
           PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=4), seed=3))
    frames = synth.sequence("S" if algo == "gmm" else "T", w, h, seed=21, frames=n)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=oracle_mod.cpu_threads())
    side = torch.cuda.Stream()
    with _engine(cfg, w, h) as eng:
        pending = None
        for t, f in enumerate(frames):
            want = ref.process_frame(f)
            kind = t % 3
            if kind == 0:  # torch tensor on a side stream, right after a submit()
                with torch.cuda.stream(side):
                    got = eng.process_frame(torch.from_numpy(f).cuda()).cpu().numpy()
                np.testing.assert_array_equal(got, want, err_msg=f"frame {t} (tensor)")
            elif kind == 1:  # numpy through the handle's stream, after a side-stream step
                np.testing.assert_array_equal(eng.process_frame(f), want,
                                              err_msg=f"frame {t} (numpy)")
            else:  # asynchronous host path, not waited for before the next step
                buf = np.empty((h, w), np.uint8)
                eng.submit(np.ascontiguousarray(f), buf)
                pending = (t, buf, want)
                continue
            if pending is not None:
                eng.synchronize()
                np.testing.assert_array_equal(pending[1], pending[2],
                                              err_msg=f"frame {pending[0]} (submit)")
                pending = None
        eng.synchronize()
        if pending is not None:
            np.testing.assert_array_equal(pending[1], pending[2], err_msg="last submit")
        torch.cuda.synchronize()
        st = {k: v for k, v in eng.state_arrays().items()}
    _assert_state_equal(st, ref.state_arrays(), list(st))


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_submit_pipelined_sequence_matches_oracle(oracle_mod, algo):
    # SegmentationEngine.submit(): frames from pinned host buffers enqueued
    # back to back with no synchronisation in between (frame t+1's upload
    # overlaps frame t's kernels and frame t-1's download, two device slots
    # per handle), then one synchronize(): every mask equals the oracle's
    # sequential run (engine.py:99-112 semantics), and so does the state.
    import torch

    w, h, n = 640, 480, 24
    cfg = (PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=7, k_d=3))
           if algo == "gmm" else
           PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=6), seed=11))
    frames = synth.sequence("S" if algo == "gmm" else "T", w, h, seed=5, frames=n)
    pinned_in = [torch.from_numpy(f).pin_memory().numpy() for f in frames]
    pinned_out = [torch.empty((h, w), dtype=torch.uint8).pin_memory().numpy() for _ in frames]
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=oracle_mod.cpu_threads())
    with _engine(cfg, w, h) as eng:
        for f, m in zip(pinned_in, pinned_out):
            eng.submit(f, m)
        eng.synchronize()
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(pinned_out[t], ref.process_frame(f), err_msg=f"frame {t}")
        # the synchronous staged path continues the same state
        for t in range(4):
            f = synth.make_frame("S" if algo == "gmm" else "T", w, h, 5, n + t)
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {n + t} (process_frame)")
        st = {k: v for k, v in eng.state_arrays().items()}
    _assert_state_equal(st, ref.state_arrays(), list(st))


@pytest.mark.parametrize("k", [3, 7])
def test_gmm_least_fit_near_ties_match_reference(oracle_mod, k):
    # Unmatched pixels replace argmin_k w_k / sqrt(v_k) (gmm.py:326-337,
    # first minimum wins).  K1 picks it from an FP32 estimate unless the
    # runner-up is within 2^-16 of the minimum (or a value is out of range);
    # these states put the exact FP64 keys at exact ties, 1-ulp and 1e-9 /
    # 1e-6 / 1e-5 / 3e-5 / 1e-3 relative gaps in every slot order, plus +0
    # weights and tiny / huge values, and check every replacement against
    # the oracle.
    rng = np.random.default_rng(17 + k)
    w_, h_ = 64, 48
    P = w_ * h_
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=k, k_d=3))
    ref = oracle_mod.OracleEngine(cfg, w_, h_, workers=1)
    ref.process_frame(synth.make_frame("T", w_, h_, 1, 0))
    st = {key: v.copy() for key, v in ref.state_arrays().items()}
    gaps = [0.0, 2.0 ** -52, 1e-9, 1e-6, 1e-5, 3e-5, 1e-3, 0.5]
    wv = np.empty((P, k))
    vv = np.empty((P, k))
    for i in range(P):
        base_f = rng.uniform(0.05, 0.3)
        v = rng.uniform(1.0, 400.0, size=k)
        f = base_f * (1.0 + rng.uniform(0.01, 1.0, size=k))  # well separated ...
        a, b = rng.choice(k, size=2, replace=False)  # ... except a near-tied pair
        g = gaps[i % len(gaps)]
        f[a] = base_f
        f[b] = base_f * (1.0 + g)
        wv[i] = f * np.sqrt(v)
        vv[i] = v
        if i % 97 == 5:  # two +0 weights (ties at 0)
            wv[i, a] = 0.0
            wv[i, b] = 0.0
        if i % 89 == 7:  # out of the FP32 estimate's range
            wv[i, a] = 1e-20
        if i % 83 == 11:
            wv[i, b] = 1e20
    st["rgb_w"] = wv.reshape(h_, w_, k)
    st["rgb_var"] = vv.reshape(h_, w_, k)
    st["rgb_mu"] = np.full((h_, w_, k, 3), 10.0)  # far from the frame below: no match
    ref.state = {key: v.copy() for key, v in st.items()}
    frame = np.zeros((h_, w_, 4), np.uint8)
    frame[..., :3] = 240
    frame[..., 3] = 0  # no depth: the RGB sub-model alone
    with _engine(cfg, w_, h_) as eng:
        eng.load_state(st)
        np.testing.assert_array_equal(eng.process_frame(frame), ref.process_frame(frame))
        got = {key: v for key, v in eng.state_arrays().items()}
    _assert_state_equal(got, ref.state_arrays(), gu.GMM_KEYS)
    # the replaced slot differs between the near-tied pair across pixels
    replaced = np.argmax(ref.state_arrays()["rgb_mu"][..., 0].reshape(P, k) == 240.0, axis=1)
    assert len(np.unique(replaced)) == k


@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_staged_host_path_row_chunks_odd_size(oracle_mod, algo):
    # process_frame(numpy) on a frame >= 4 MB runs the row-chunked staged
    # path (csrc/common.cuh HostStaging::run_rows): chunk i segments while
    # chunk i+1 is staged by the helper threads.  An odd width makes the PBAS
    # chunks align to 32 rows (list-mode row launches start on 32-pixel
    # boundaries) and leaves a ragged last chunk; masks and state must equal
    # the oracle, and a numpy frame mixed with a CUDA-tensor frame stays ordered.
    import torch

    w, h, n = 1283, 833, 14
    assert 4 * w * h >= 4 << 20
    cfg = (PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams(k_rgb=4, k_d=2))
           if algo == "gmm" else
           PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(n=4), seed=17))
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=oracle_mod.cpu_threads())
    with _engine(cfg, w, h) as eng:
        for t in range(n):
            f = synth.make_frame("T", w, h, 31, t)
            want = ref.process_frame(f)
            if t == 9:
                got = eng.process_frame(torch.from_numpy(f).cuda()).cpu().numpy()
            else:
                got = eng.process_frame(f)
            np.testing.assert_array_equal(got, want, err_msg=f"frame {t}")
        st = {k: v for k, v in eng.state_arrays().items()}
    _assert_state_equal(st, ref.state_arrays(), list(st))
