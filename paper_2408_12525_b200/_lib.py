"""ctypes binding of the C ABI in include/pcgrl_b200.h.

The CUDA library is the product path: there is no CPU fallback. If the
shared object is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LG_LIB_PATH") or os.path.join(_PKG, "libpcgrl_b200.so")  # override: experiments

LG_OK, LG_EINVAL, LG_ECUDA = 0, 1, 2
FLAG_BAD_ACTION, FLAG_NO_EDITABLE, FLAG_PINPOINTS = 1, 2, 4
STEP_NO_AUTO_RESET = 1
STEP_VALIDATE = 2

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


class LgConfig(ctypes.Structure):
    _fields_ = [
        ("domain", ctypes.c_int32), ("representation", ctypes.c_int32),
        ("max_h", ctypes.c_int32), ("max_w", ctypes.c_int32),
        ("obs_size", ctypes.c_int32), ("randomize_shape", ctypes.c_int32),
        ("init_weighted", ctypes.c_int32), ("n_pins", ctypes.c_int32),
        ("pins", ctypes.c_int32 * 16), ("n_ctrl", ctypes.c_int32),
        ("ctrl", ctypes.c_int32 * 8), ("max_steps", ctypes.c_int64),
        ("change_budget", ctypes.c_int64), ("det_metrics", ctypes.c_int32),
        ("obs_format", ctypes.c_int32), ("init_cdf", ctypes.c_double * 8),
        ("weights", ctypes.c_double * 8),
    ]


class LgInfo(ctypes.Structure):
    _fields_ = [(n, _P) for n in ("terminal", "episode_reward", "episode_length",
                                  "episode_start_loss", "final_loss")]


STATE_FIELDS = ("tiles", "active", "frozen", "shape_hw", "order", "order_len", "pos_idx", "pos",
                "t", "changes", "max_steps", "lo", "hi", "values", "unreach", "prev_loss",
                "ep_reward", "ep_start_loss", "metric_seeds", "rng")


class LgState(ctypes.Structure):
    _fields_ = [(n, _P) for n in STATE_FIELDS]


class LgDesc(ctypes.Structure):
    _fields_ = [("n_envs", ctypes.c_int64), ("n_actions", ctypes.c_int32),
                ("n_metrics", ctypes.c_int32), ("obs_c", ctypes.c_int32),
                ("obs_h", ctypes.c_int32), ("obs_w", ctypes.c_int32), ("team", ctypes.c_int32),
                ("obs_bytes_per_env", ctypes.c_int64), ("state_bytes_per_env", ctypes.c_int64)]


# every symbol include/pcgrl_b200.h declares, with its ctypes signature
SIGNATURES = {
    "lg_last_error": (ctypes.c_char_p, []),
    "lg_version": (ctypes.c_char_p, []),
    "lg_create": (ctypes.c_int, [ctypes.POINTER(LgConfig), _I64, _I64, ctypes.c_uint64, ctypes.c_int,
                                 ctypes.POINTER(_P)]),
    "lg_destroy": (ctypes.c_int, [_P]),
    "lg_describe": (ctypes.c_int, [_P, ctypes.POINTER(LgDesc)]),
    "lg_reset": (ctypes.c_int, [_P, _P, _P]),
    "lg_reset_masked": (ctypes.c_int, [_P, _P, _P, _P]),
    "lg_step": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.POINTER(LgInfo), _P, _P]),
    "lg_step_flags": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.POINTER(LgInfo), _P, ctypes.c_uint32,
                                     _P]),
    "lg_observe": (ctypes.c_int, [_P, _P, _P]),
    "lg_recompute": (ctypes.c_int, [_P, _P, ctypes.c_int, _P]),
    "lg_step_host": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.POINTER(LgInfo), _P]),
    "lg_export_state": (ctypes.c_int, [_P, ctypes.POINTER(LgState), _P]),
    "lg_import_state": (ctypes.c_int, [_P, ctypes.POINTER(LgState), _P]),
    "lg_errors": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint32), _P]),
    "lg_random_actions": (ctypes.c_int, [_P, _P, ctypes.c_uint64, _P]),
    "lg_step_random": (ctypes.c_int, [_P, ctypes.c_uint64, _P, _P, _P, _P, ctypes.POINTER(LgInfo), _P, _P]),
    "lg_first_episode": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P]),
    "lg_metrics": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I64, _P, _P, _P, _P, _P,
                                  _P]),
    "lg_seed_streams": (ctypes.c_int, [ctypes.c_uint64, _I64, _I64, _P]),
    "lg_policy_trunk": (ctypes.c_int, [_P, _I64, ctypes.c_int, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P, _P]),
    "lg_policy_trunk_sample": (ctypes.c_int, [_P, _I64, ctypes.c_int, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P,
                                              ctypes.c_uint64, _P, _P, _P]),
    "lg_host_threads": (ctypes.c_int, []),
    "lg_unpack_host": (ctypes.c_int, [_P, _I64, _P, ctypes.c_int]),
    "lg_conv1_bits": (ctypes.c_int, [_P, _I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_int,
                                     _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA extension {path} is missing; build it with "
            "`python -m paper_2408_12525_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("LG_LIB_PATH") and not hasattr(lib, name):
            continue  # an older variant build (LG_LIB_PATH A/B runs): entry points it predates
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == LG_OK:
        return
    msg = load().lg_last_error().decode()
    if rc == LG_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)
