"""ctypes binding of the C ABI (include/voltyard_b200.h).

The CUDA library is mandatory: if ``libvoltyard_b200.so`` is missing or fails
to load, every entry point raises ``NativeError`` — there is no CPU fallback
in the product path.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import EpisodeDone, NativeError

LIB_PATH = Path(__file__).resolve().parent / "libvoltyard_b200.so"

VY_OK, VY_ERR_ARG, VY_ERR_CUDA, VY_ERR_UNSUPPORTED, VY_ERR_STATE = 0, 1, 2, 3, 4
VY_ACT_U8, VY_ACT_I32, VY_ACT_I64 = 0, 1, 2
COLSUM_BANDS = 2048  # VY_COLSUM_BANDS
F_AUTO_RESET, F_INFOS, F_INJECT, F_OUT_F64 = 1, 2, 4, 8

_P = C.c_void_p


class VyState(C.Structure):
    _fields_ = [("ld", C.c_int64)] + [(n, _P) for n in (
        "port_i", "port_soc", "port_de", "port_dtrem", "port_meta", "step", "day", "episode", "env_seed", "akey",
        "b_i", "b_soc", "ep_profit", "ep_reward", "ep_missing", "ep_energy", "ep_overtime", "ep_declined",
        "ep_departures")]


class VyOutputs(C.Structure):
    _fields_ = [(n, _P) for n in (
        "obs", "reward", "done", "ep_stats", "term_overtime", "breakdown", "flows", "declined", "arrivals_m",
        "dep_n", "dep_port", "dep_overtime", "dep_early", "dep_pref", "dep_missing", "dep_cap", "dep_soc",
        "i_att", "i_used", "delivered", "b_delivered")]


class VyDraws(C.Structure):
    _fields_ = [(n, _P) for n in ("off", "profile", "stay", "soc0", "frac", "pref")]


_lib: C.CDLL | None = None

# name -> (restype, argtypes); mirrors include/voltyard_b200.h
_SIGS = {
    "vy_abi_version": (C.c_int, []),
    "vy_last_error": (C.c_char_p, []),
    "vy_create": (C.c_int, [_P, C.c_int64, C.c_int, C.POINTER(_P)]),
    "vy_destroy": (C.c_int, [_P]),
    "vy_add_profile": (C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_double]),
    "vy_get_profile": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double)]),
    "vy_bind": (C.c_int, [_P, C.POINTER(VyState), C.POINTER(VyOutputs)]),
    "vy_reset": (C.c_int, [_P, _P, C.c_int32, _P, C.c_uint32, _P]),
    "vy_reset_episodes": (C.c_int, [_P, _P, _P, C.c_uint32, _P]),
    "vy_seed_envs": (C.c_int, [_P, C.c_int64, C.c_int64, _P]),
    "vy_step": (C.c_int, [_P, _P, C.c_int32, C.c_int64, C.c_int64, C.c_uint32, C.POINTER(VyDraws), _P]),
    "vy_random_actions": (C.c_int, [_P, C.c_uint64, C.c_int64, C.c_int64, _P, _P]),
    "vy_random_actions_dev": (C.c_int, [_P, C.c_uint64, C.c_int64, _P, _P, _P]),
    "vy_step_random": (C.c_int, [_P, C.c_uint64, C.c_int64, C.c_int64, _P, _P, C.c_uint32, _P]),
    "vy_rollout": (C.c_int, [_P, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, _P, C.c_int64, _P, _P, C.c_int64,
                             C.c_uint32, _P]),
    "vy_poll_error": (C.c_int, [_P, C.c_int, _P, C.POINTER(C.c_uint32)]),
    "vy_launch_count": (C.c_int64, [_P]),
    "vy_last_step_mode": (C.c_int32, [_P]),
    "vy_set_tiles_per_warp": (C.c_int, [_P, C.c_int32]),
    "vy_set_wide": (C.c_int, [_P, C.c_int32]),
    "vy_gae": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_int64, C.c_float, C.c_float, _P, _P, _P]),
    "vy_ppo_sample": (C.c_int, [_P, C.c_int32, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]),
    "vy_ppo_sample_rng": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_uint64, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P,
                                    _P, C.c_int32, _P]),
    "vy_ppo_head_fwd": (C.c_int, [_P, C.c_int32, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P]),
    "vy_ppo_head_bwd": (C.c_int, [_P, C.c_int32, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P,
                                  C.c_int32, _P, _P]),
    "vy_gather_rows": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _P, _P]),
    "vy_colsum": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_int64, C.c_int64, _P, _P, _P]),
    "vy_policy_geometry": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
    "vy_policy_step": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _P, _P, C.c_uint64, _P,
                                 _P, _P, _P, _P, _P]),
    "vy_ppo_rollout": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int32, C.c_int32, C.c_uint64, _P, _P, _P, _P, _P, _P, _P,
                                 _P]),
    "vy_ppo_update_workspace": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                          C.POINTER(C.c_int64)]),
    "vy_ppo_update_grad": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64, _P, _P, _P,
                                     _P, C.c_int64, C.c_float, C.c_float, C.c_float, C.c_float, _P, _P, _P, _P, _P]),
    "vy_ppo_update_adam": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _P, _P, _P, _P, _P,
                                     _P, C.c_float, C.c_float, C.c_float, C.c_float, _P]),
    "vy_ppo_adv_stats": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.c_int64, _P, _P]),
    "vy_gae_scal": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int64, C.c_float, C.c_float, _P, _P]),
    "vy_random_perms": (C.c_int, [C.c_int64, C.c_int32, C.c_uint64, _P, _P, _P]),
    "vy_selftest_div": (C.c_int, [C.POINTER(C.c_double), C.c_int32, C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]),
    "vy_ppo_loss": (C.c_int, [_P, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P, C.c_float, C.c_float,
                              C.c_float, C.c_float, C.c_int32, _P, _P, _P]),
    "vy_scale_bf16": (C.c_int, [_P, C.c_int64, _P, _P]),
    "vy_multi_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.POINTER(C.c_uint64), C.POINTER(C.c_int64),
                                  C.POINTER(_P)]),
    "vy_multi_step_random": (C.c_int, [_P, C.c_int64, _P, _P]),
    "vy_multi_info": (C.c_int32, [_P, C.POINTER(C.c_int32)]),
    "vy_multi_launch_count": (C.c_int64, [_P]),
    "vy_multi_destroy": (C.c_int, [_P]),
}


def exported_symbols() -> tuple[str, ...]:
    return tuple(_SIGS)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(f"CUDA extension not built: {LIB_PATH} missing (run __graft_entry__.build())")
        try:
            handle = C.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise NativeError(f"failed to load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc == VY_OK:
        return
    msg = f"{what}: {lib().vy_last_error().decode()}"
    if rc == VY_ERR_ARG:
        raise ValueError(msg)
    if rc == VY_ERR_STATE:
        raise EpisodeDone(msg)
    if rc == VY_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(msg)
