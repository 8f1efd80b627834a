"""ctypes binding of libgridrogue_b200.so (include/gridrogue_b200.h).

This is the only way the Python layer reaches the compute path.  There is
no fallback: if the library is missing or no CUDA device is present, the
calls fail loudly.
"""

from __future__ import annotations

import ctypes
import os

from ._build import LIB

GR_OK = 0
GR_E_INVALID = -1
GR_E_CUDA = -2
GR_E_STATE = -3
GR_E_BAD_ACTION = -4
GR_E_OOM = -5

TIER_IDS = {"classic": 0, "extended": 1}
OBS_IDS = {"none": 0, "symbolic": 1, "pixels": 2}

# state field ids == gridrogue.state.FIELD_NAMES order (state.py:29-125)
FIELD_NAMES = (
    "blocks", "items", "ladder_down", "ladder_up", "spawn0", "potion_map", "chest_pos",
    "chest_loot", "chest_qty", "chest_aux", "necro_pos", "params_seed", "pfloor", "prow",
    "pcol", "facing", "health", "food", "drink", "energy", "mana", "xp", "dex", "str_",
    "intel", "sword_tier", "pick_tier", "has_bow", "sword_ench", "bow_ench", "armour",
    "armour_ench", "learned_fire", "learned_ice", "sleeping", "resting", "inv_wood",
    "inv_stone", "inv_coal", "inv_iron", "inv_diamond", "inv_sapphire", "inv_ruby",
    "inv_sapling", "inv_torch", "inv_arrow", "inv_book", "inv_potion", "mel_pos", "mel_hp",
    "mel_cd", "mel_alive", "mel_type", "ran_pos", "ran_hp", "ran_cd", "ran_alive",
    "ran_type", "pas_pos", "pas_hp", "pas_alive", "pas_type", "pproj_pos", "pproj_dir",
    "pproj_type", "pproj_ttl", "pproj_alive", "pproj_dmg", "eproj_pos", "eproj_dir",
    "eproj_type", "eproj_ttl", "eproj_alive", "eproj_dmg", "plant_pos", "plant_age",
    "plant_alive", "ach", "time", "rng_key", "floors_visited", "floor_cleared", "boss_hp",
    "boss_wave", "boss_vuln", "boss_timer", "clocks", "done",
)
FIELD_ID = {n: i for i, n in enumerate(FIELD_NAMES)}


class GrConfig(ctypes.Structure):
    _fields_ = [
        ("tier", ctypes.c_int32), ("obs_mode", ctypes.c_int32), ("tile_px", ctypes.c_int32),
        ("reset_ratio", ctypes.c_int32), ("n_envs", ctypes.c_int64), ("env_offset", ctypes.c_int64),
        ("n_envs_global", ctypes.c_int64), ("max_episode_length", ctypes.c_int64),
        ("seed", ctypes.c_uint64), ("device", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


class GrStats(ctypes.Structure):
    _fields_ = [("episodes", ctypes.c_int64), ("total_steps", ctypes.c_int64),
                ("total_return", ctypes.c_double), ("ach_episodes", ctypes.c_int64 * 67)]


class GridrogueError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    # GR_LIB_VARIANT=name loads lib/ab/name.so instead (A/B timing of two
    # builds in one process tree on one box; still the in-tree CUDA library)
    path = LIB
    variant = os.environ.get("GR_LIB_VARIANT")
    if variant:
        path = os.path.join(os.path.dirname(LIB), "ab", variant + ".so")
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: the CUDA extension has not been built "
            "(run `python -m paper_2402_16801_b200._build` or __graft_entry__.build()); "
            "there is no CPU fallback")
    L = ctypes.CDLL(path)
    P, I32, I64, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    sig = {
        "gr_create": (I32, [ctypes.POINTER(GrConfig), ctypes.POINTER(P)]),
        "gr_destroy": (None, [P]),
        "gr_last_error": (ctypes.c_char_p, []),
        "gr_version": (I32, []),
        "gr_obs_elems": (I64, [P]),
        "gr_n_actions": (I32, [P]),
        "gr_n_achievements": (I32, [P]),
        "gr_field_info": (I32, [I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I32)]),
        "gr_reset": (I32, [P, P, P]),
        "gr_step": (I32, [P, P, P, P, P, P, P, P, P]),
        "gr_random_actions": (I32, [P, ctypes.c_uint32, U64, P, P]),
        "gr_set_validate": (I32, [P, I32]),
        "gr_bad_action": (I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "gr_step_local": (I32, [P, P, P, P, P, P, P, P, P]),
        "gr_step_finish": (I32, [P, P, I32, I32, P, P]),
        "gr_step_host": (I32, [P, P, P, P, P, P, P, P]),
        "gr_reset_host": (I32, [P, P]),
        "gr_host_obs_attach": (I32, [P, P]),
        "gr_host_obs_detach": (I32, [P, P]),
        "gr_host_phase_times": (I32, [P, P, P, P]),
        "gr_obs_to_host": (I32, [P, P, P, P]),
        "gr_account_replay": (I32, [P, I64, I64]),
        "gr_export_field": (I32, [P, I32, P]),
        "gr_import_field": (I32, [P, I32, P]),
        "gr_observe": (I32, [P, P, P]),
        "gr_stats_get": (I32, [P, ctypes.POINTER(GrStats)]),
        "gr_stats_set": (I32, [P, ctypes.POINTER(GrStats)]),
        "gr_level_seeds": (I32, [P, P]),
        "gr_episodes_completed": (I32, [P, ctypes.POINTER(I64)]),
        "gr_export_episode": (I32, [P, P, P]),
        "gr_levels_create": (I32, [P, I64, ctypes.POINTER(P)]),
        "gr_levels_destroy": (None, [P]),
        "gr_levels_set_params": (I32, [P, I64, I64, P, P, P]),
        "gr_levels_get_params": (I32, [P, I64, I64, P, P, P]),
        "gr_levels_generate": (I32, [P, I64, I64]),
        "gr_levels_mutate": (I32, [P, I32, I64, P, P, P, ctypes.c_double]),
        "gr_levels_install": (I32, [P, I64, P, P, P]),
        "gr_levels_export_world": (I32, [P, I64, P, P, P, P, P, P]),
        "gr_levels_world_info": (I32, [P, I64, P, P]),
        "gr_levels_import_world": (I32, [P, I64, U64, P, P, P, P, P, P, ctypes.c_uint32]),
        "gr_import_episode": (I32, [P, P, P]),
        "gr_get_step_index": (I32, [P, ctypes.POINTER(I64)]),
        "gr_set_step_index": (I32, [P, I64]),
        "gr_kernel_launches": (I64, [P]),
        "gr_worldgen_counters": (I32, [P, ctypes.POINTER(I64)]),
        "gr_set_worldgen_attempts": (I32, [P, I32]),
        "gr_selftest_sincos64": (I32, [P, P, P, I64, P]),
        "gr_selftest_argsort6": (I32, [P, P, I64, P]),
        "gr_set_profiling": (I32, [P, I32]),
        "gr_kernel_times": (I32, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64), I32]),
        # include/gridrogue_ppo.h (the learner's fused objective)
        "grp_ppo_loss": (I32, [P, P, P, P, P, P, P, I32, I32, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                               P, P, P, P]),
        "grp_sample_actions": (I32, [P, P, I32, I32, I32, I64, I64, U64, P, ctypes.c_uint32, P, P, P, P, P, P,
                                     P, P, P]),
        "grp_ppo_loss_bf16": (I32, [P, I64, P, I64, P, P, P, P, P, I32, I32, ctypes.c_float, ctypes.c_float,
                                    ctypes.c_float, P, I64, I32, P, I64, P, P, P]),
        "grp_bias_grad": (I32, [P, I64, P, I64, P, I64, I32, I32, I32, P, P, P, I32, P, I32, I64, I64, I64, P]),
        "grp_bias_tanh": (I32, [P, P, I32, I32, I32, P]),
        "grp_rows_to_bf16": (I32, [P, I64, I32, P, I64, P]),
        "grp_clip_adam": (I32, [P, P, P, P, P, I64, P, P, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                ctypes.c_float, ctypes.c_float, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != GR_OK:
        msg = lib().gr_last_error().decode(errors="replace")
        if rc == GR_E_INVALID or rc == GR_E_BAD_ACTION:
            raise ValueError(msg)
        if rc == GR_E_STATE:
            raise RuntimeError(msg)
        raise GridrogueError(f"gridrogue_b200 error {rc}: {msg}")
