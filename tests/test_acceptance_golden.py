"""The reference's acceptance criteria 3 and 7 (tests/test_acceptance.py:
125-139, :200-233), pinned on the CPU side: the fixtures in
tests/golden/accept_c*.npz were produced by the reference engine itself
(tests/golden/make_golden.py).  Here: the scene generator restated in
synth.py reproduces the reference's input frames, and the oracle
(the parity checker of the device path) reproduces the reference's masks,
invariants and final state.  The device side is tests/test_gpu_acceptance.py."""

import hashlib

import numpy as np

import golden_util as gu
from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import PipelineConfig


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def criterion3_frames():
    """tests/test_acceptance.py:128-134: 500 noisy 64x64 frames, depth valid."""
    rng = np.random.default_rng(99)
    for _ in range(500):
        frame = rng.integers(0, 256, size=(64, 64, 4), dtype=np.uint8)
        frame[:, :, 3] = rng.integers(1, 256, size=(64, 64))
        yield frame


def criterion7_spec():
    return synth.SceneSpec("colour_camouflage", width=160, height=120, frames=200,
                           entry_frame=100)


def test_criterion7_scene_inputs_equal_reference():
    fx = gu.load("accept_c7.npz")
    spec = criterion7_spec()
    for t in range(spec.frames):
        rgb, d16, _ = synth.scene_frame(spec, t)
        assert _sha(rgb) == fx["rgb_sha"][t], f"rgb frame {t}"
        assert _sha(d16) == fx["d16_sha"][t], f"depth frame {t}"


def test_oracle_criterion3_invariants_masks_state(oracle_mod):
    fx = gu.load("accept_c3.npz")
    ref = oracle_mod.OracleEngine(PipelineConfig(algorithm="gmm", mode="rgbd"), 64, 64, workers=2)
    for t, frame in enumerate(criterion3_frames()):
        m = ref.process_frame(frame)
        np.testing.assert_array_equal(np.packbits(m > 0), fx["masks"][t], err_msg=f"frame {t}")
        st = ref.state_arrays()
        dev = max(float(np.abs(st[k].sum(axis=2) - 1.0).max()) for k in ("rgb_w", "d_w"))
        vmin = min(float(st[k].min()) for k in ("rgb_var", "d_var"))
        assert dev <= 1e-9 and vmin >= 1.0, (t, dev, vmin)
        assert dev == fx["wsum_dev"][t] and vmin == fx["var_min"][t], t
    st = ref.state_arrays()
    assert [_sha(st[k]) for k in fx["state_keys"]] == list(fx["state_sha"])


def test_oracle_criterion7_masks_and_state(oracle_mod):
    fx = gu.load("accept_c7.npz")
    spec = criterion7_spec()
    frames = [oracle_mod.pack_frame(*synth.scene_frame(spec, t)[:2]) for t in range(spec.frames)]
    assert [_sha(f) for f in frames] == list(fx["frame_sha"])
    for algo in ("gmm", "pbas"):
        ref = oracle_mod.OracleEngine(PipelineConfig(algorithm=algo, mode="rgbd", seed=42),
                                      160, 120, workers=4)
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(np.packbits(ref.process_frame(f) > 0),
                                          fx[f"{algo}_masks"][t], err_msg=f"{algo} frame {t}")
        st = ref.state_arrays()
        assert [_sha(st[k]) for k in fx[f"{algo}_state_keys"]] == list(fx[f"{algo}_state_sha"]), algo
