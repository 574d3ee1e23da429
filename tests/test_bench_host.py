"""Host-side logic of bench.py that runs without a GPU: the clock sampler's
nvidia-smi fallback parsing, the throttle rule (hw / thermal slowdown is
re-measured, sw_power_cap is kept) and the B_alg table the roofline uses."""

import bench


def test_throttle_rule_single_rank():
    assert not bench._throttled(None, None, 1)
    assert not bench._throttled({"reasons": ["sw_power_cap"]}, None, 1)
    for r in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"):
        assert bench._throttled({"reasons": [r, "sw_power_cap"]}, None, 1)


def test_clock_sampler_parses_nvidia_smi_rows(tmp_path):
    # the nvidia-smi fallback: index, sm, max sm, power, 4 reason columns
    s = bench.ClockSampler(0)
    f = tmp_path / "clk.csv"
    f.write_text("0, 1965, 1965, 700.1, Not Active, Not Active, Not Active, Active\n"
                 "0, 1890, 1965, 710.0, Not Active, Not Active, Not Active, Not Active\n"
                 "garbage line\n")

    class _Done:
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

        def kill(self):
            pass

    class _F:
        name = str(f)

        def flush(self):
            pass

    s.proc, s.f = _Done(), _F()
    out = s.stop()
    assert out["samples"] == 2 and out["source"] == "nvidia-smi"
    assert out["sm_max_mhz"] == 1965 and out["sm_mhz"] == (1965 + 1890) / 2
    assert out["reasons"] == ["sw_power_cap"]


def test_b_alg_table_matches_survey():
    # GMM 7/3 485, 3/3 293, PBAS n=20 181, f32-storage GMM 7/3 245 B/px
    assert bench.B_ALG[("gmm", 7, 3)] == 485
    assert bench.B_ALG[("gmm", 3, 3)] == 293
    assert bench.B_ALG[("pbas", 20)] == 181
    assert bench.B_ALG[("gmm_f32", 7, 3)] == 245
    # f32: half of the 352 + 128 state bytes + 5 frame/mask bytes; 3/3: (192 + 96) / 2 + 5
    assert bench.B_ALG[("gmm_f32", 3, 3)] == (192 + 96) // 2 + 5


def test_bit_equality_folds_are_position_weighted_and_match_torch():
    # bench._fold_np / _fold_dev: position-weighted 64-bit folds (wrapping),
    # the cross-rank bit-equality proof of config 5 and the stream digests
    import numpy as np
    import torch

    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, size=1003, dtype=np.uint8)
    words = np.concatenate([a, np.zeros((-a.size) % 8, np.uint8)]).view(np.uint64)
    want = sum(int(w) * (2 * i + 1) for i, w in enumerate(words)) % (1 << 64)
    assert bench._fold_np(a) == want
    # torch's int64 fold is the same number modulo 2^64
    assert bench._fold_dev(torch.from_numpy(a)) % (1 << 64) == want
    b = a.copy()
    b[[0, 8]] = b[[8, 0]]  # same bytes, different positions
    assert bench._fold_np(b) != bench._fold_np(a) or a[0] == a[8]
    assert bench._mix(bench._mix(0, 1), 2) != bench._mix(bench._mix(0, 2), 1)
