"""Opt-in PBAS gradient feature (config.PbasGradient) -- the CPU side.

The feature is NOT in the reference (SPEC.md:314 omits the original PBAS
gradient term), so its checker is this package's own restatement,
oracle_pbas_frame_g (oracle/rgbdseg_oracle.c).  That restatement is pinned
here three ways:
  * its Sobel magnitude map equals an independent numpy statement;
  * at alpha = 0 the term vanishes, so masks and every reference state array
    must equal the plain restatement (itself pinned to the reference's golden
    vectors, test_oracle_golden.py) bit for bit;
  * on small grids a pure-Python per-pixel statement of the whole frame
    (classification, rings, R/T, RNG, self/neighbour updates) agrees exactly.
"""

import math

import numpy as np
import pytest

from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import PbasGradient, PbasParams, PipelineConfig
from paper_2002_00250_b200.errors import ConfigError
from paper_2002_00250_b200.config import validate_config


def _cfg(n=6, mm=2, mode="rgbd", seed=5, grad=PbasGradient()):
    return PipelineConfig(algorithm="pbas", mode=mode, pbas=PbasParams(n=n, min_matches=mm),
                          seed=seed, pbas_gradient=grad)


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (6, 1), (2, 2), (13, 37), (40, 33)])
def test_gradient_map_matches_numpy(oracle_mod, shape):
    h, w = shape
    rng = np.random.default_rng(h * 100 + w)
    frame = rng.integers(0, 256, size=(h, w, 4), dtype=np.uint8)
    g, total = oracle_mod.gradient_map(frame)
    want = oracle_mod.gradient_map_np(frame)
    np.testing.assert_array_equal(g, want)
    assert total == int(want.astype(np.int64).sum())


def test_gradient_map_extremes(oracle_mod):
    # a vertical step 0 | 255 reaches the top magnitude 4*255 per axis (>> 3 = 127)
    frame = np.zeros((5, 6, 4), dtype=np.uint8)
    frame[:, 3:, :3] = 255
    g = oracle_mod.gradient_map_np(frame)
    assert g.max() == (4 * 255) >> 3
    # a checkerboard drives |Sx| + |Sy| to its maximum 2040 -> 255
    cb = ((np.indices((8, 8)).sum(axis=0) % 2) * 255).astype(np.uint8)
    frame = np.repeat(cb[:, :, None], 4, axis=2)
    g2, _ = oracle_mod.gradient_map(frame)
    np.testing.assert_array_equal(g2, oracle_mod.gradient_map_np(frame))
    assert g2.max() <= 255


@pytest.mark.parametrize("mode,mm,n", [("rgbd", 2, 6), ("rgb_only", 1, 5), ("rgbd", 3, 9)])
def test_alpha_zero_equals_reference_restatement(oracle_mod, mode, mm, n):
    w, h = 29, 17
    frames = synth.sequence("T", w, h, seed=3, frames=n + 25)
    plain = oracle_mod.OracleEngine(_cfg(n, mm, mode, grad=None), w, h, workers=2)
    grad = oracle_mod.OracleEngine(_cfg(n, mm, mode, grad=PbasGradient(alpha=0.0)), w, h, workers=3)
    for t, f in enumerate(frames):
        np.testing.assert_array_equal(grad.process_frame(f), plain.process_frame(f), err_msg=f"frame {t}")
    for k, v in plain.state_arrays().items():
        np.testing.assert_array_equal(grad.state_arrays()[k], v, err_msg=k)
    # the per-sample magnitudes are still tracked
    assert grad.state_arrays()["samples_grad"].any()


def test_gradient_changes_the_decision(oracle_mod):
    w, h, n = 40, 24, 6
    frames = synth.sequence("T", w, h, seed=9, frames=n + 30)
    plain = oracle_mod.OracleEngine(_cfg(n, grad=None), w, h, workers=1)
    grad = oracle_mod.OracleEngine(_cfg(n, grad=PbasGradient(alpha=10.0)), w, h, workers=1)
    diff = 0
    for f in frames:
        diff += int(np.count_nonzero(grad.process_frame(f) != plain.process_frame(f)))
    assert diff > 0
    # the previous-frame sum is carried as state
    assert int(grad.state_arrays()["grad_prev_sum"]) == oracle_mod.gradient_map(frames[-1])[1]


# ---------------------------------------------------------------- pure Python
_NBR = [(-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1)]


def _py_frame(oracle_mod, st, frame, f, cfg, prev_sum):
    """One frame of PBAS with the gradient feature, pixel by pixel in Python
    (the reference's _pbas_band, pbas.py:344-508, plus the feature's terms),
    intents applied after the scan (pbas.py:511-522)."""
    p, g = cfg.pbas, cfg.pbas_gradient
    h, w = frame.shape[:2]
    n = p.n
    use_depth = cfg.mode == "rgbd"
    gmap = oracle_mod.gradient_map_np(frame).astype(int)
    mean = g.mean_init if prev_sum is None else prev_sum / (h * w)
    wt = min(65535, int(math.floor(g.alpha * 256.0 / (mean if mean > 1.0 else 1.0) + 0.5)))
    mask = np.zeros((h, w), np.uint8)
    intents = []
    S, G = st["samples"], st["samples_grad"]
    for y in range(h):
        for x in range(w):
            r, gg, b = (int(v) for v in frame[y, x, :3])
            d = int(frame[y, x, 3]) if use_depth else 0
            gm = int(gmap[y, x])
            if f < n:
                S[y, x, f] = (r, gg, b, d)
                G[y, x, f] = gm
                continue
            cnt, dmin256 = 0, 255 * 256
            for i in range(n):
                sr, sg, sb, _ = (int(v) for v in S[y, x, i])
                dist = max(abs(r - sr), abs(gg - sg), abs(b - sb))
                dd = 256 * dist + wt * abs(gm - int(G[y, x, i]))
                cnt += dd < 256 * st["r_rgb"][y, x]  # exact: int vs a power-of-two multiple
                dmin256 = min(dmin256, dd)
            dminr = dmin256 >> 8
            bg_rgb = cnt >= p.min_matches
            depth_eval, bg_depth, dmind = False, True, 255
            if d > 0:
                valid = cntd = 0
                for i in range(n):
                    sd = int(S[y, x, i, 3])
                    if sd == 0:
                        continue
                    valid += 1
                    dist = abs(d - sd)
                    cntd += float(dist) < st["r_d"][y, x]
                    dmind = min(dmind, dist)
                if valid >= p.min_matches:
                    depth_eval, bg_depth = True, cntd >= p.min_matches
            fg = (not bg_rgb) or (depth_eval and not bg_depth)
            mask[y, x] = 255 if fg else 0

            def ring(kind, val, rkey):
                ringv, pos, ln = st["dmin_" + kind][y, x], st["pos_" + kind], st["len_" + kind]
                ringv[pos[y, x]] = val
                pos[y, x] = (int(pos[y, x]) + 1) % n
                if ln[y, x] < n:
                    ln[y, x] += 1
                avg = float(int(ringv[: ln[y, x]].astype(np.int64).sum())) / float(ln[y, x])
                rv = st[rkey][y, x]
                rv = rv * (1.0 - p.r_inc_dec) if rv > avg * p.r_scale else rv * (1.0 + p.r_inc_dec)
                st[rkey][y, x] = max(rv, p.r_lower) if rv < p.r_lower else rv
                return avg

            avg_rgb = ring("rgb", dminr, "r_rgb")
            if depth_eval:
                ring("d", dmind, "r_d")
            guard = avg_rgb if avg_rgb > 1.0 else 1.0
            t = st["t"][y, x] + (p.t_inc / guard if fg else -(p.t_dec / guard))
            st["t"][y, x] = min(max(t, p.t_lower), p.t_upper)
            if fg:
                continue
            prob = 1.0 / st["t"][y, x]
            seed = cfg.seed
            u0 = oracle_mod.pixel_rng_py(seed, x, y, f, 0)
            if u0 < prob:
                slot = min(int((u0 / prob) * n), n - 1)
                S[y, x, slot] = (r, gg, b, d)
                G[y, x, slot] = gm
            u1 = oracle_mod.pixel_rng_py(seed, x, y, f, 1)
            if u1 < prob:
                inb = [(y + dy, x + dx) for dy, dx in _NBR if 0 <= y + dy < h and 0 <= x + dx < w]
                pick = min(int((u1 / prob) * len(inb)), len(inb) - 1)
                u2 = oracle_mod.pixel_rng_py(seed, x, y, f, 2)
                intents.append((*inb[pick], min(int(u2 * n), n - 1)))
    for ny, nx, slot in intents:
        S[ny, nx, slot] = (*frame[ny, nx, :3], frame[ny, nx, 3] if use_depth else 0)
        G[ny, nx, slot] = gmap[ny, nx]
    return mask, int(gmap.sum())


def test_gradient_weight(oracle_mod):
    none = oracle_mod.GRAD_NONE
    assert oracle_mod.gradient_weight(none, 100, 10.0, 20.0) == 128  # 2560 / 20
    assert oracle_mod.gradient_weight(2000, 100, 10.0, 20.0) == 128  # mean 20
    assert oracle_mod.gradient_weight(0, 100, 10.0, 20.0) == 2560    # mean floored at 1
    assert oracle_mod.gradient_weight(0, 100, 1e9, 20.0) == 65535    # capped
    assert oracle_mod.gradient_weight(0, 100, 0.0, 20.0) == 0
    assert oracle_mod.gradient_weight(300, 100, 1.0, 20.0) == 85     # 256/3 = 85.33


@pytest.mark.parametrize("mode,alpha,seed", [("rgbd", 10.0, 11), ("rgb_only", 3.5, 12)])
def test_c_restatement_matches_pure_python(oracle_mod, mode, alpha, seed):
    w, h, n = 9, 7, 4
    cfg = _cfg(n, 2, mode, seed=seed, grad=PbasGradient(alpha=alpha, mean_init=15.0))
    frames = synth.sequence("T", w, h, seed=seed, frames=n + 14)
    eng = oracle_mod.OracleEngine(cfg, w, h, workers=2)
    st = {k: np.array(v, copy=True) for k, v in eng.state_arrays().items()}
    prev = None
    for t, f in enumerate(frames):
        want, prev = _py_frame(oracle_mod, st, f, t, cfg, prev)
        got = eng.process_frame(f)
        if t >= n:
            np.testing.assert_array_equal(got, want, err_msg=f"frame {t}")
    for k, v in eng.state_arrays().items():
        if k != "grad_prev_sum":
            np.testing.assert_array_equal(v, st[k], err_msg=k)
    assert int(eng.state_arrays()["grad_prev_sum"]) == prev


def test_config_validation():
    validate_config(_cfg())
    for bad in (PbasGradient(alpha=-1.0), PbasGradient(alpha=float("nan")),
                PbasGradient(mean_init=0.0), PbasGradient(mean_init=float("inf"))):
        with pytest.raises(ConfigError):
            validate_config(_cfg(grad=bad))
