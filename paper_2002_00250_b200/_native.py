"""ctypes binding of the C-ABI (include/rgbdseg_b200.h).

Loads the in-tree librgbdseg_b200.so built by `_build.build()`.  There is no
fallback: if the library is missing or fails to load, `lib()` raises
DeviceError.  Status codes map onto the reference's exception classes
(errors.py:4-21): 1 -> DimensionError, 2 -> ConfigError, 3 -> DeviceError
(an RgbdSegError).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError, DeviceError, DimensionError

LIB_PATH = Path(os.environ.get("RGBDSEG_B200_LIB") or
                Path(__file__).resolve().parent / "librgbdseg_b200.so")

# Every symbol include/rgbdseg_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "rgbdseg_last_error", "rgbdseg_abi_version", "rgbdseg_device_count",
    "rgbdseg_rng_stream", "rgbdseg_rng_keys",
    "rgbdseg_gmm_create", "rgbdseg_gmm_create_ex", "rgbdseg_gmm_destroy", "rgbdseg_gmm_step", "rgbdseg_gmm_step_batch",
    "rgbdseg_gmm_process_host", "rgbdseg_gmm_sync", "rgbdseg_gmm_state_bytes",
    "rgbdseg_gmm_read_state", "rgbdseg_gmm_write_state", "rgbdseg_gmm_stream",
    "rgbdseg_pbas_create", "rgbdseg_pbas_create_band", "rgbdseg_pbas_destroy",
    "rgbdseg_pbas_step", "rgbdseg_pbas_classify", "rgbdseg_pbas_apply", "rgbdseg_pbas_halo_ptrs",
    "rgbdseg_pbas_classify_rows", "rgbdseg_pbas_copy_edges", "rgbdseg_pbas_set_halos",
    "rgbdseg_pbas_step_batch", "rgbdseg_pbas_process_host", "rgbdseg_pbas_sync",
    "rgbdseg_pbas_get_frame_idx", "rgbdseg_pbas_set_frame_idx", "rgbdseg_pbas_state_bytes",
    "rgbdseg_pbas_read_state", "rgbdseg_pbas_write_state", "rgbdseg_pbas_stream",
    "rgbdseg_confusion_accumulate", "rgbdseg_pack_frame", "rgbdseg_median3x3",
    "rgbdseg_halo_link_create", "rgbdseg_halo_link_export", "rgbdseg_halo_link_connect",
    "rgbdseg_halo_link_connect_local", "rgbdseg_halo_link_push", "rgbdseg_halo_link_pull",
    "rgbdseg_halo_link_set_timeout", "rgbdseg_halo_link_status", "rgbdseg_halo_link_error",
    "rgbdseg_halo_link_destroy",
    "rgbdseg_selftest_fdiv", "rgbdseg_gmm_set_eval", "rgbdseg_gmm_eval_counts",
    "rgbdseg_pbas_set_eval", "rgbdseg_pbas_eval_counts", "rgbdseg_pbas_set_k2_mode",
    "rgbdseg_pbas_get_k2_mode", "rgbdseg_pbas_set_gradient",
)

IPC_HANDLE_BYTES = 64  # RGBDSEG_IPC_HANDLE_BYTES

GMM_STATE_F32 = 1  # RGBDSEG_GMM_STATE_F32
GMM_FIELDS = {"rgb_w": 0, "rgb_mu": 1, "rgb_var": 2, "d_w": 3, "d_mu": 4, "d_var": 5}
PBAS_FIELDS = {"samples": 0, "dmin_rgb": 1, "dmin_d": 2, "len_rgb": 3, "pos_rgb": 4,
               "len_d": 5, "pos_d": 6, "r_rgb": 7, "r_d": 8, "t": 9,
               # opt-in gradient feature (config.PbasGradient) only
               "samples_grad": 10, "grad_prev_sum": 11}


class GmmParamsC(ctypes.Structure):
    _fields_ = [("k_rgb", ctypes.c_int32), ("k_d", ctypes.c_int32), ("alpha", ctypes.c_double),
                ("s", ctypes.c_double), ("tau", ctypes.c_double),
                ("match_lambda", ctypes.c_double), ("var_init", ctypes.c_double),
                ("w_init", ctypes.c_double)]


class PbasParamsC(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("min_matches", ctypes.c_int32),
                ("r_init", ctypes.c_double), ("r_lower", ctypes.c_double),
                ("r_scale", ctypes.c_double), ("r_inc_dec", ctypes.c_double),
                ("t_init", ctypes.c_double), ("t_lower", ctypes.c_double),
                ("t_upper", ctypes.c_double), ("t_inc", ctypes.c_double),
                ("t_dec", ctypes.c_double)]


_lib = None


def _declare(L):
    vp, i32, i64, u64, f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                              ctypes.c_double)
    P = ctypes.POINTER
    sig = {
        "rgbdseg_last_error": (ctypes.c_char_p, []),
        "rgbdseg_abi_version": (i32, []),
        "rgbdseg_device_count": (i32, []),
        "rgbdseg_rng_stream": (ctypes.c_int, [u64, u64, u64, u64, i64, vp, i32]),
        "rgbdseg_rng_keys": (ctypes.c_int, [vp, i64, vp, i32]),
        "rgbdseg_gmm_create": (ctypes.c_int, [i32, i32, P(GmmParamsC), i32, i32, P(vp)]),
        "rgbdseg_gmm_create_ex": (ctypes.c_int, [i32, i32, P(GmmParamsC), i32, i32, ctypes.c_uint32,
                                                 P(vp)]),
        "rgbdseg_gmm_destroy": (None, [vp]),
        "rgbdseg_gmm_step": (ctypes.c_int, [vp, vp, vp, vp]),
        "rgbdseg_gmm_step_batch": (ctypes.c_int, [vp, i32, vp, vp, vp]),
        "rgbdseg_gmm_process_host": (ctypes.c_int, [vp, vp, vp, i32]),
        "rgbdseg_gmm_sync": (ctypes.c_int, [vp]),
        "rgbdseg_gmm_state_bytes": (i64, [vp, i32]),
        "rgbdseg_gmm_read_state": (ctypes.c_int, [vp, i32, vp, i64]),
        "rgbdseg_gmm_write_state": (ctypes.c_int, [vp, i32, vp, i64]),
        "rgbdseg_gmm_stream": (vp, [vp]),
        "rgbdseg_pbas_create": (ctypes.c_int, [i32, i32, P(PbasParamsC), i32, u64, i32, P(vp)]),
        "rgbdseg_pbas_create_band": (ctypes.c_int,
                                     [i32, i32, i32, i32, P(PbasParamsC), i32, u64, i32, P(vp)]),
        "rgbdseg_pbas_destroy": (None, [vp]),
        "rgbdseg_pbas_step": (ctypes.c_int, [vp, vp, vp, vp]),
        "rgbdseg_pbas_classify": (ctypes.c_int, [vp, vp, vp, vp]),
        "rgbdseg_pbas_apply": (ctypes.c_int, [vp, vp, vp]),
        "rgbdseg_pbas_halo_ptrs": (ctypes.c_int, [vp, P(vp), P(vp), P(vp), P(vp), P(i64)]),
        "rgbdseg_pbas_classify_rows": (ctypes.c_int, [vp, vp, vp, i32, i32, vp]),
        "rgbdseg_pbas_copy_edges": (ctypes.c_int, [vp, vp, vp, vp]),
        "rgbdseg_pbas_set_halos": (ctypes.c_int, [vp, vp, vp, vp]),
        "rgbdseg_pbas_step_batch": (ctypes.c_int, [vp, i32, vp, vp, vp]),
        "rgbdseg_pbas_process_host": (ctypes.c_int, [vp, vp, vp, i32]),
        "rgbdseg_pbas_sync": (ctypes.c_int, [vp]),
        "rgbdseg_pbas_get_frame_idx": (u64, [vp]),
        "rgbdseg_pbas_set_frame_idx": (ctypes.c_int, [vp, u64]),
        "rgbdseg_pbas_state_bytes": (i64, [vp, i32]),
        "rgbdseg_pbas_read_state": (ctypes.c_int, [vp, i32, vp, i64]),
        "rgbdseg_pbas_write_state": (ctypes.c_int, [vp, i32, vp, i64]),
        "rgbdseg_pbas_stream": (vp, [vp]),
        "rgbdseg_confusion_accumulate": (ctypes.c_int, [vp, vp, i64, vp, vp]),
        "rgbdseg_pack_frame": (ctypes.c_int, [vp, i32, i32, vp, i32, i32, vp, vp]),
        "rgbdseg_median3x3": (ctypes.c_int, [vp, vp, i32, i32, vp]),
        "rgbdseg_halo_link_create": (ctypes.c_int, [vp, i32, P(vp)]),
        "rgbdseg_halo_link_export": (ctypes.c_int, [vp, vp]),
        "rgbdseg_halo_link_connect": (ctypes.c_int, [vp, vp, vp]),
        "rgbdseg_halo_link_connect_local": (ctypes.c_int, [vp, vp, vp]),
        "rgbdseg_halo_link_push": (ctypes.c_int, [vp, u64, vp]),
        "rgbdseg_halo_link_pull": (ctypes.c_int, [vp, u64, vp]),
        "rgbdseg_halo_link_set_timeout": (ctypes.c_int, [vp, u64]),
        "rgbdseg_halo_link_status": (ctypes.c_int, [vp]),
        "rgbdseg_halo_link_error": (i32, [vp]),
        "rgbdseg_halo_link_destroy": (None, [vp]),
        "rgbdseg_selftest_fdiv": (ctypes.c_int, [vp, vp, i64, P(i64)]),
        "rgbdseg_gmm_set_eval": (ctypes.c_int, [vp, vp]),
        "rgbdseg_gmm_eval_counts": (ctypes.c_int, [vp, vp, i32, i32, vp]),
        "rgbdseg_pbas_set_eval": (ctypes.c_int, [vp, vp]),
        "rgbdseg_pbas_eval_counts": (ctypes.c_int, [vp, vp, i32, i32, vp]),
        "rgbdseg_pbas_set_k2_mode": (ctypes.c_int, [vp, i32]),
        "rgbdseg_pbas_get_k2_mode": (i32, [vp]),
        "rgbdseg_pbas_set_gradient": (ctypes.c_int, [vp, i32, ctypes.c_double, ctypes.c_double]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded C-ABI library (raises DeviceError when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if os.environ.get("RGBDSEG_B200_AUTOBUILD", "1") == "1":
            from . import _build

            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - surfaced below
                raise DeviceError(f"native extension missing and build failed: {exc}") from exc
        if not LIB_PATH.exists():
            raise DeviceError(f"native extension {LIB_PATH} is missing; run __graft_entry__.build()")
    try:
        L = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    _declare(L)
    _lib = L
    return L


def last_error() -> str:
    msg = lib().rgbdseg_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = last_error()
    text = f"{what}: {msg}" if what else msg
    if rc == 1:
        raise DimensionError(text)
    if rc == 2:
        raise ConfigError(text)
    raise DeviceError(text)


def device_count() -> int:
    return int(lib().rgbdseg_device_count())


def gmm_params_c(p) -> GmmParamsC:
    return GmmParamsC(int(p.k_rgb), int(p.k_d), float(p.alpha), float(p.s), float(p.tau),
                      float(p.match_lambda), float(p.var_init), float(p.w_init))


def pbas_params_c(p) -> PbasParamsC:
    return PbasParamsC(int(p.n), int(p.min_matches), float(p.r_init), float(p.r_lower),
                       float(p.r_scale), float(p.r_inc_dec), float(p.t_init), float(p.t_lower),
                       float(p.t_upper), float(p.t_inc), float(p.t_dec))
