"""CPU-only checks of the C-ABI boundary: the library loads, exports every
symbol include/rgbdseg_b200.h declares, and maps status codes onto the
reference's exception classes (errors.py:4-21) -- no compute calls."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2002_00250_b200 import _build, _native
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig
from paper_2002_00250_b200.errors import ConfigError, DeviceError, DimensionError, RgbdSegError

HEADER = Path(__file__).resolve().parent.parent / "include" / "rgbdseg_b200.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rgbdseg_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_for_sm100a():
    lib = _build.build()
    assert lib.exists()


def test_exports_every_declared_symbol():
    L = _native.lib()
    declared = header_functions()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_native.EXPORTS)


def test_abi_version_and_device_count():
    L = _native.lib()
    assert L.rgbdseg_abi_version() == 1
    assert _native.device_count() >= 0


def test_config_errors_before_device():
    L = _native.lib()
    h = ctypes.c_void_p()
    bad = _native.gmm_params_c(GmmParams(k_rgb=0))
    assert L.rgbdseg_gmm_create(4, 4, ctypes.byref(bad), 1, 0, ctypes.byref(h)) == 2
    assert "component counts" in _native.last_error()
    good = _native.gmm_params_c(GmmParams())
    assert L.rgbdseg_gmm_create(0, 4, ctypes.byref(good), 1, 0, ctypes.byref(h)) == 1
    badp = _native.pbas_params_c(PbasParams(n=1, min_matches=2))
    assert L.rgbdseg_pbas_create(4, 4, ctypes.byref(badp), 1, 0, 0, ctypes.byref(h)) == 2
    bigp = _native.pbas_params_c(PbasParams(n=300))
    assert L.rgbdseg_pbas_create(4, 4, ctypes.byref(bigp), 1, 0, 0, ctypes.byref(h)) == 2
    okp = _native.pbas_params_c(PbasParams())
    assert L.rgbdseg_pbas_create_band(4, 4, 3, 2, ctypes.byref(okp), 1, 0, 0,
                                      ctypes.byref(h)) == 1


def test_status_code_mapping():
    with pytest.raises(DimensionError):
        _native.check(1)
    with pytest.raises(ConfigError):
        _native.check(2)
    with pytest.raises(DeviceError):
        _native.check(3)
    assert issubclass(DeviceError, RgbdSegError)


def test_engine_validates_like_reference():
    # ConfigError from PipelineConfig.validate (config.py:37-50), then
    # DimensionError (engine.py:62-63), before any device work.
    from paper_2002_00250_b200.engine import SegmentationEngine

    with pytest.raises(ConfigError):
        SegmentationEngine(PipelineConfig(algorithm="sift"), 4, 4)
    with pytest.raises(ConfigError):
        SegmentationEngine(PipelineConfig(mode="depth"), 4, 4)
    with pytest.raises(ConfigError):
        SegmentationEngine(PipelineConfig(gmm=GmmParams(alpha=0)), 4, 4)
    with pytest.raises(ConfigError):
        SegmentationEngine(PipelineConfig(pbas=PbasParams(t_init=500)), 4, 4)
    with pytest.raises(ConfigError):
        SegmentationEngine(PipelineConfig(seed=2 ** 64), 4, 4)
    with pytest.raises(DimensionError):
        SegmentationEngine(PipelineConfig(), 0, 4)


@pytest.mark.skipif(_native.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_silent_cpu_fallback():
    from paper_2002_00250_b200.engine import SegmentationEngine

    with pytest.raises(DeviceError):
        SegmentationEngine(PipelineConfig(), 8, 6)


def _udiv_magic(d):
    """Python twin of csrc/common.cuh udiv_magic/udiv (Granlund-Montgomery)."""
    if d <= 1:
        return 0, 0
    l = (d - 1).bit_length()
    return ((1 << 32) * ((1 << l) - d)) // d + 1, l


def _udiv(n, d):
    m, l = _udiv_magic(d)
    if l == 0:
        return n
    t = (n * m) >> 32
    return (t + ((n - t) >> 1)) >> (l - 1)


def test_magic_division_used_for_pixel_rows():
    # K2 maps pixel index -> (row, column) with this 32-bit magic division.
    import numpy as np

    rng = np.random.default_rng(0)
    widths = list(range(1, 3000)) + [7680, 3840, 1920, 1280, 640, 2 ** 31 - 1]
    for d in widths:
        m, _ = _udiv_magic(d)
        assert m < 2 ** 32
        ns = [0, 1, d - 1, d, d + 1, 2 ** 31 - 1] + [int(v) for v in rng.integers(0, 2 ** 31, 20)]
        for n in ns:
            assert _udiv(n, d) == n // d, (n, d)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["gmm", "pbas"])
def test_plain_c_host_matches_python_engine(tmp_path, algo):
    # examples/capi_demo.c drives the path through the C-ABI alone (the
    # boundary a non-Python host binds); its masks and state must equal the
    # Python engine's on the same frames, bit for bit.
    import subprocess

    import numpy as np

    from paper_2002_00250_b200 import _build
    from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig
    from paper_2002_00250_b200.engine import SegmentationEngine

    exe = _build.build_capi_demo()
    w, h, n, seed = 64, 48, 30, 7
    out = tmp_path / "demo.bin"
    subprocess.run([str(exe), algo, str(w), str(h), str(n), str(seed), str(out)], check=True)
    raw = np.fromfile(out, dtype=np.uint8)
    frames = raw[: n * h * w * 4].reshape(n, h, w, 4)
    masks = raw[n * h * w * 4: n * h * w * 5].reshape(n, h, w)
    state = raw[n * h * w * 5:].view(np.float64)
    cfg = (PipelineConfig(algorithm="gmm", mode="rgbd", gmm=GmmParams()) if algo == "gmm" else
           PipelineConfig(algorithm="pbas", mode="rgbd", pbas=PbasParams(), seed=seed + 1))
    with SegmentationEngine(cfg, w, h, device=0) as eng:
        for t in range(n):
            np.testing.assert_array_equal(eng.process_frame(frames[t]), masks[t], err_msg=f"frame {t}")
        key = "rgb_w" if algo == "gmm" else "r_rgb"
        np.testing.assert_array_equal(eng.state_arrays()[key].ravel(), state)
