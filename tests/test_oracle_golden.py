"""Pin the CPU restatement (oracle/) against the reference's own outputs.

The fixtures were produced by the reference (tests/golden/make_golden.py):
its pure-Python oracle tests/reference.py for the *_equiv_* cases and its
numba SegmentationEngine for the synthetic sequences.  Bit-exact masks and
state are required, exactly as the reference's TestKernelEquivalence
(tests/test_gmm.py:222-248, tests/test_pbas.py:463-491) requires of its
kernels.  Also carries over the reference's scalar known-answer tests
(tests/test_gmm.py:36-219, tests/test_pbas.py:27-188) restated on 1-pixel
grids.
"""

import math

import numpy as np
import pytest

import golden_util as gu
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig


@pytest.mark.parametrize("name", gu.gmm_cases())
@pytest.mark.parametrize("workers", [1, 3])
def test_oracle_gmm_matches_reference(oracle_mod, name, workers):
    fx = gu.load(name)
    cfg = gu.gmm_config(fx, name)
    frames = fx["frames"]
    eng = oracle_mod.OracleEngine(cfg, frames.shape[2], frames.shape[1], workers=workers)
    for t, f in enumerate(frames):
        np.testing.assert_array_equal(eng.process_frame(f), fx["masks"][t], err_msg=f"frame {t}")
    st = eng.state_arrays()
    for k in gu.GMM_KEYS:
        np.testing.assert_array_equal(st[k], fx[k], err_msg=k)


@pytest.mark.parametrize("name", gu.pbas_cases())
@pytest.mark.parametrize("workers", [1, 4])
def test_oracle_pbas_matches_reference(oracle_mod, name, workers):
    fx = gu.load(name)
    cfg = gu.pbas_config(fx, name)
    frames = fx["frames"]
    eng = oracle_mod.OracleEngine(cfg, frames.shape[2], frames.shape[1], workers=workers)
    for t, f in enumerate(frames):
        np.testing.assert_array_equal(eng.process_frame(f), fx["masks"][t], err_msg=f"frame {t}")
    st = eng.state_arrays()
    for k in gu.PBAS_KEYS:
        np.testing.assert_array_equal(st[k], fx[k], err_msg=k)


def test_oracle_rng_matches_reference(oracle_mod):
    fx = gu.load("rng.npz")
    for key, val in zip(fx["keys"], fx["values"]):
        k = [int(v) for v in key]
        assert oracle_mod.pixel_rng(*k) == val
        assert oracle_mod.pixel_rng_py(*k) == val
    s, x, y, f = (int(v) for v in fx["stream_key"])
    np.testing.assert_array_equal(oracle_mod.rng_stream(s, x, y, f, len(fx["stream"])), fx["stream"])


# ----- scalar known-answer tests, restated through one-pixel grids ---------

def _gmm1(oracle_mod, params, rgb_comps, d_comps=(), mode="rgb_only"):
    cfg = PipelineConfig(algorithm="gmm", mode=mode, gmm=params)
    eng = oracle_mod.OracleEngine(cfg, 1, 1)
    st = eng.state_arrays()
    for k, (w, mu, v) in enumerate(rgb_comps):
        st["rgb_w"][0, 0, k] = w
        st["rgb_mu"][0, 0, k] = mu
        st["rgb_var"][0, 0, k] = v
    for k, (w, mu, v) in enumerate(d_comps):
        st["d_w"][0, 0, k] = w
        st["d_mu"][0, 0, k] = mu
        st["d_var"][0, 0, k] = v
    return eng


def _px(rgb, d=0):
    return np.array([[[rgb[0], rgb[1], rgb[2], d]]], dtype=np.uint8)


def test_kat_weight_recurrence(oracle_mod):
    # tests/test_gmm.py:143-150
    eng = _gmm1(oracle_mod, GmmParams(k_rgb=2, alpha=0.001),
                [(0.5, [0, 0, 0], 100.0), (0.5, [200, 200, 200], 100.0)])
    eng.process_frame(_px((0, 0, 0)))
    w = eng.state_arrays()["rgb_w"][0, 0]
    assert w[0] == pytest.approx(0.5005, abs=1e-12)
    assert w[1] == pytest.approx(0.4995, abs=1e-12)


def test_kat_least_fit_replacement(oracle_mod):
    # tests/test_gmm.py:165-177
    params = GmmParams(k_rgb=3, w_init=0.05, var_init=225.0)
    eng = _gmm1(oracle_mod, params, [(0.6, [0, 0, 0], 100.0), (0.1, [50, 50, 50], 400.0),
                                      (0.3, [200, 200, 200], 100.0)])
    eng.process_frame(_px((120, 120, 120)))
    st = eng.state_arrays()
    assert st["rgb_mu"][0, 0, 1].tolist() == [120.0, 120.0, 120.0]
    assert st["rgb_var"][0, 0, 1] == 225.0
    assert st["rgb_w"][0, 0].sum() == pytest.approx(1.0, abs=1e-12)
    assert st["rgb_w"][0, 0, 1] == pytest.approx(0.05 / (0.6 + 0.1 + 0.3 - 0.1 + 0.05), rel=1e-9)


def test_kat_blend(oracle_mod):
    # tests/test_gmm.py:179-186
    eng = _gmm1(oracle_mod, GmmParams(k_rgb=1, alpha=0.5), [(1.0, [10, 10, 10], 16.0)])
    eng.process_frame(_px((12, 10, 10)))
    st = eng.state_arrays()
    assert st["rgb_mu"][0, 0, 0].tolist() == [11.0, 10.0, 10.0]
    assert st["rgb_var"][0, 0, 0] == pytest.approx(0.5 * 16.0 + 0.5 * 4.0)


def test_kat_first_frame_background_and_depth_seed(oracle_mod):
    # tests/test_gmm.py:203-219: first frame seeds and is background; the
    # depth mixture seeds on its first valid reading.
    cfg = PipelineConfig(algorithm="gmm", mode="rgbd")
    eng = oracle_mod.OracleEngine(cfg, 1, 1)
    assert eng.process_frame(_px((40, 80, 120), 200))[0, 0] == 0
    eng2 = oracle_mod.OracleEngine(cfg, 1, 1)
    eng2.process_frame(_px((1, 2, 3), 0))
    assert eng2.state_arrays()["d_w"][0, 0, 0] == 0.0
    eng2.process_frame(_px((1, 2, 3), 77))
    assert eng2.state_arrays()["d_w"][0, 0, 0] == 1.0
    assert eng2.state_arrays()["d_mu"][0, 0, 0, 0] == 77.0


def test_kat_depth_mismatch_is_foreground(oracle_mod):
    # tests/test_gmm.py:110-120: depth far off collapses the product below tau
    eng = _gmm1(oracle_mod, GmmParams(), [(1.0, [10, 20, 30], 100.0)], [(1.0, [100], 100.0)],
                mode="rgbd")
    assert eng.process_frame(_px((10, 20, 30), 250))[0, 0] == 255
    s = 10000.0
    p_rgb = s / (2.0 * math.pi * 100.0)
    p_d = p_rgb * math.exp(-(150.0 ** 2 / 200.0))
    assert p_rgb * p_d < 1.0


def _pbas1(oracle_mod, params, sample, mode="rgbd", seed=0, frame_idx=None):
    cfg = PipelineConfig(algorithm="pbas", mode=mode, pbas=params, seed=seed)
    eng = oracle_mod.OracleEngine(cfg, 1, 1)
    eng.state_arrays()["samples"][0, 0, :] = sample
    eng.frame_idx = params.n if frame_idx is None else frame_idx
    return eng


def test_kat_pbas_camouflage_caught_by_depth(oracle_mod):
    # tests/test_pbas.py:322-330
    eng = _pbas1(oracle_mod, PbasParams(), (10, 20, 30, 150))
    assert eng.process_frame(_px((10, 20, 30), 90))[0, 0] == 255
    assert eng.state_arrays()["dmin_d"][0, 0, 0] == 60


def test_kat_pbas_invalid_depth_gates_to_rgb(oracle_mod):
    # tests/test_pbas.py:332-345
    eng = _pbas1(oracle_mod, PbasParams(), (10, 20, 30, 150))
    assert eng.process_frame(_px((10, 20, 30), 0))[0, 0] == 0
    eng = _pbas1(oracle_mod, PbasParams(), (10, 20, 30, 0))
    eng.state_arrays()["samples"][0, 0, 0, 3] = 200
    assert eng.process_frame(_px((10, 20, 30), 90))[0, 0] == 0
    assert eng.state_arrays()["len_d"][0, 0] == 0  # depth abstained


def test_kat_pbas_R_and_T_adaptation(oracle_mod):
    # tests/test_pbas.py:361-409: R grows 18 -> 18.9 when R <= 5*avg;
    # T drops by t_dec/guard on background.
    eng = _pbas1(oracle_mod, PbasParams(), (10, 20, 30, 40))
    eng.process_frame(_px((20, 20, 30), 40))  # rgb dist 10 to every sample -> avg 10
    st = eng.state_arrays()
    assert st["r_rgb"][0, 0] == pytest.approx(18.9, abs=1e-12)
    assert st["t"][0, 0] == pytest.approx(18.0 - 0.05 / 10.0, abs=1e-12)


def test_oracle_pack_frame_matches_reference(oracle_mod):
    # frames.pack_frame(rgb, resample_depth(d16, W, H)) produced by the reference
    fx = gu.load("frames.npz")
    for tag in ("all", "up", "odd", "down", "p720_480"):
        np.testing.assert_array_equal(oracle_mod.pack_frame(fx[f"{tag}_rgb"], fx[f"{tag}_d16"]),
                                      fx[f"{tag}_frame"], err_msg=tag)


def test_markstein_ratio_exhaustive(tmp_path):
    # K2's ratio() (csrc/pbas.cu) replaces the IEEE divide tot / len of the
    # dmin averages (pbas.py:432, :448) by a Markstein step with RN(1/n):
    # exact for every (tot, len) the state can hold.
    import shutil
    import subprocess
    from pathlib import Path

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = Path(__file__).parent / "native" / "markstein_ratio.c"
    exe = tmp_path / "markstein_ratio"
    subprocess.run([cc, "-O2", "-ffp-contract=off", "-o", str(exe), str(src), "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "cases 16711680 mismatches 0" in r.stdout
