"""B200-native RGB-D foreground segmentation (depth-extended GMM + PBAS).

Drop-in for the reference `rgbdseg` engine path (pkg/src/rgbdseg/engine.py):
`SegmentationEngine(config, width, height)`, `.process_frame(frame)`,
`.state_arrays()`.  The per-pixel work runs in hand-written sm_100a CUDA
kernels (csrc/) behind a C-ABI (include/rgbdseg_b200.h); there is no CPU
fallback — a missing extension raises `DeviceError`.
"""

from .config import GmmParams, PbasGradient, PbasParams, PipelineConfig
from .errors import (
    ConfigError,
    DeviceError,
    DimensionError,
    FormatError,
    RgbdSegError,
    SequenceError,
)

__version__ = "0.1.0"

_LAZY = {
    "SegmentationEngine": ("engine", "SegmentationEngine"),
    "MultiStreamEngine": ("engine", "MultiStreamEngine"),
    "pixel_rng": ("rng", "pixel_rng"),
    "rng_stream": ("rng", "rng_stream"),
    "process_sequence": ("sequence", "process_sequence"),
    "RunStats": ("sequence", "RunStats"),
    "MemorySequence": ("sequence", "MemorySequence"),
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod, attr = _LAZY[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)


__all__ = [
    "GmmParams", "PbasGradient", "PbasParams", "PipelineConfig", "SegmentationEngine", "MultiStreamEngine",
    "pixel_rng", "rng_stream", "process_sequence", "RunStats", "MemorySequence", "RgbdSegError",
    "DimensionError", "FormatError",
    "SequenceError", "ConfigError", "DeviceError", "__version__",
]
