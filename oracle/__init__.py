"""CPU oracle for the gridrogue batched-env hot path -- TEST INFRASTRUCTURE.

A ctypes wrapper over ``oracle/build/libgr_oracle.so`` (plain C restatement
of the numpy reference, see ``gr_oracle.h``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` leg may import this package: it is the checker, never the thing
measured or shipped.  The product (``paper_2402_16801_b200``) does not import
it and fails loudly when its own CUDA library is missing.

State arrays use the reference's SimState layout and field order
(``/root/reference/pkg/src/gridrogue/state.py:29-125``), so a reference
SimState can be imported field by field and compared bit for bit.
"""

from __future__ import annotations

import ctypes
import os
import shutil
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libgr_oracle.so")

# (name, dtype, trailing template) -- state.py:29-125, same order
FIELDS = [
    ("blocks", np.uint8, ("F", "H", "W")), ("items", np.uint8, ("F", "H", "W")),
    ("ladder_down", np.int16, ("F", 2)), ("ladder_up", np.int16, ("F", 2)),
    ("spawn0", np.int16, (2,)), ("potion_map", np.uint8, (6,)),
    ("chest_pos", np.int16, ("F", 6, 2)), ("chest_loot", np.uint8, ("F", 6)),
    ("chest_qty", np.uint8, ("F", 6)), ("chest_aux", np.uint8, ("F", 6)),
    ("necro_pos", np.int16, (2,)), ("params_seed", np.uint64, ()),
    ("pfloor", np.uint8, ()), ("prow", np.int16, ()), ("pcol", np.int16, ()),
    ("facing", np.uint8, ()), ("health", np.float32, ()), ("food", np.float32, ()),
    ("drink", np.float32, ()), ("energy", np.float32, ()), ("mana", np.float32, ()),
    ("xp", np.uint8, ()), ("dex", np.uint8, ()), ("str_", np.uint8, ()),
    ("intel", np.uint8, ()), ("sword_tier", np.uint8, ()), ("pick_tier", np.uint8, ()),
    ("has_bow", np.bool_, ()), ("sword_ench", np.uint8, ()), ("bow_ench", np.uint8, ()),
    ("armour", np.uint8, (4,)), ("armour_ench", np.uint8, (4,)),
    ("learned_fire", np.bool_, ()), ("learned_ice", np.bool_, ()),
    ("sleeping", np.bool_, ()), ("resting", np.bool_, ()),
    ("inv_wood", np.uint8, ()), ("inv_stone", np.uint8, ()), ("inv_coal", np.uint8, ()),
    ("inv_iron", np.uint8, ()), ("inv_diamond", np.uint8, ()),
    ("inv_sapphire", np.uint8, ()), ("inv_ruby", np.uint8, ()),
    ("inv_sapling", np.uint8, ()), ("inv_torch", np.uint8, ()),
    ("inv_arrow", np.uint8, ()), ("inv_book", np.uint8, ()),
    ("inv_potion", np.uint8, (6,)),
    ("mel_pos", np.int16, ("F", 3, 2)), ("mel_hp", np.float32, ("F", 3)),
    ("mel_cd", np.uint8, ("F", 3)), ("mel_alive", np.bool_, ("F", 3)),
    ("mel_type", np.uint8, ("F", 3)),
    ("ran_pos", np.int16, ("F", 2, 2)), ("ran_hp", np.float32, ("F", 2)),
    ("ran_cd", np.uint8, ("F", 2)), ("ran_alive", np.bool_, ("F", 2)),
    ("ran_type", np.uint8, ("F", 2)),
    ("pas_pos", np.int16, ("F", 3, 2)), ("pas_hp", np.float32, ("F", 3)),
    ("pas_alive", np.bool_, ("F", 3)), ("pas_type", np.uint8, ("F", 3)),
    ("pproj_pos", np.int16, (3, 2)), ("pproj_dir", np.uint8, (3,)),
    ("pproj_type", np.uint8, (3,)), ("pproj_ttl", np.uint8, (3,)),
    ("pproj_alive", np.bool_, (3,)), ("pproj_dmg", np.float32, (3, 3)),
    ("eproj_pos", np.int16, (3, 2)), ("eproj_dir", np.uint8, (3,)),
    ("eproj_type", np.uint8, (3,)), ("eproj_ttl", np.uint8, (3,)),
    ("eproj_alive", np.bool_, (3,)), ("eproj_dmg", np.float32, (3, 3)),
    ("plant_pos", np.int16, (10, 2)), ("plant_age", np.uint16, (10,)),
    ("plant_alive", np.bool_, (10,)),
    ("ach", np.bool_, ("A",)), ("time", np.uint32, ()), ("rng_key", np.uint64, ()),
    ("floors_visited", np.bool_, ("F",)), ("floor_cleared", np.bool_, ("F",)),
    ("boss_hp", np.float32, ()), ("boss_wave", np.uint8, ()), ("boss_vuln", np.bool_, ()),
    ("boss_timer", np.uint8, ()), ("clocks", np.uint16, (6,)), ("done", np.bool_, ()),
]
FIELD_NAMES = tuple(f[0] for f in FIELDS)

TIERS = {
    "classic": dict(classic=1, F=1, H=64, W=64, A=22, NA=17, VR=7, VC=9, L=1345),
    "extended": dict(classic=0, F=9, H=48, W=48, A=67, NA=43, VR=9, VC=11, L=8268),
}


def field_shapes(tier: str, n: int) -> dict:
    t = TIERS[tier]
    dims = {"F": t["F"], "H": t["H"], "W": t["W"], "A": t["A"]}
    return {name: (dt, (n,) + tuple(dims.get(d, d) for d in tr)) for name, dt, tr in FIELDS}


def alloc_fields(tier: str, n: int) -> dict:
    return {k: np.zeros(shape, dt) for k, (dt, shape) in field_shapes(tier, n).items()}


def pixel_shape(tier: str, px: int) -> tuple:
    t = TIERS[tier]
    side = 0 if t["classic"] else 2
    return ((t["VR"] + 2) * px, (t["VC"] + side) * px, 3)


def build(force: bool = False) -> str:
    """Compile the oracle library (gcc, plain C, -ffp-contract=off)."""
    if shutil.which("make") is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError("make not found and the oracle library is not built")
        return _LIB_PATH
    subprocess.run(["make", "-s", "-C", _HERE] + (["-B"] if force else []), check=True)   # incremental
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        c = ctypes
        P = c.c_void_p
        L.go_hash2.restype = c.c_uint64
        L.go_hash2.argtypes = [c.c_uint64, c.c_uint64]
        L.go_mix.restype = c.c_uint64
        L.go_mix.argtypes = [c.c_uint64]
        L.go_vuniform32.restype = c.c_float
        L.go_vuniform32.argtypes = [c.c_uint32, c.c_uint32]
        L.go_np_sinf.restype = c.c_float
        L.go_np_sinf.argtypes = [c.c_float]
        L.go_np_cosf.restype = c.c_float
        L.go_np_cosf.argtypes = [c.c_float]
        L.go_np_argsort6.argtypes = [P, P]
        L.go_set_max_gen_retries.argtypes = [c.c_int]
        L.go_level_angles.argtypes = [c.c_uint64, P, P]
        L.go_generate_world.argtypes = [c.c_uint64, c.c_int, P]
        L.go_state_new.restype = P
        L.go_state_new.argtypes = [c.c_int, c.c_int64, c.c_int64]
        L.go_state_free.argtypes = [P]
        L.go_state_import.argtypes = [P, P]
        L.go_state_export.argtypes = [P, P]
        L.go_state_install_seed.argtypes = [P, c.c_int64, c.c_uint64, c.c_uint64]
        L.go_state_step.restype = c.c_int64
        L.go_state_step.argtypes = [P, P, P, P, P, P]
        L.go_state_encode.argtypes = [P, P]
        L.go_state_pixels.argtypes = [P, c.c_int, P]
        L.go_batch_create.restype = P
        L.go_batch_create.argtypes = [c.c_int, c.c_int64, c.c_uint64, c.c_int, c.c_int64, c.c_int]
        L.go_batch_destroy.argtypes = [P]
        L.go_batch_state.restype = P
        L.go_batch_state.argtypes = [P]
        L.go_batch_step.restype = c.c_int64
        L.go_batch_step.argtypes = [P, P, P, P, P, P, P]
        L.go_batch_stats.argtypes = [P, P, P, P, P]
        L.go_batch_ep.argtypes = [P, P, P]
        L.go_random_actions.argtypes = [c.c_uint32, c.c_uint64, c.c_int64, c.c_int64, c.c_int, P]
        L.go_batch_create_shard.restype = P
        L.go_batch_create_shard.argtypes = [c.c_int, c.c_int64, c.c_int64, c.c_int64, c.c_uint64, c.c_int,
                                            c.c_int64, c.c_int]
        L.go_batch_step_a.restype = c.c_int64
        L.go_batch_step_a.argtypes = [P, P, P]
        L.go_batch_step_b.restype = c.c_int64
        L.go_batch_step_b.argtypes = [P, P, P, P, P, P, P]
        L.go_batch_step_c.argtypes = [P, c.c_int64]
        L.go_state_any_dark.restype = c.c_int
        L.go_state_any_dark.argtypes = [P]
        L.go_state_encode_flag.argtypes = [P, c.c_int, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class _World(ctypes.Structure):
    _fields_ = [("blocks", ctypes.c_uint8 * (9 * 4096)), ("items", ctypes.c_uint8 * (9 * 4096)),
                ("spawn", ctypes.c_int16 * 2), ("ladder_down", ctypes.c_int16 * 18),
                ("ladder_up", ctypes.c_int16 * 18), ("chest", ctypes.c_int16 * (9 * 6 * 4)),
                ("n_chests", ctypes.c_int32 * 9), ("potion", ctypes.c_uint8 * 6),
                ("seed", ctypes.c_uint64), ("attempts", ctypes.c_int32 * 9),
                ("potion_tie", ctypes.c_int32)]


def generate_world(seed: int, tier: str) -> dict:
    """worldgen.generate_world(make_level_params(seed), tier) as arrays."""
    t = TIERS[tier]
    w = _World()
    lib().go_generate_world(ctypes.c_uint64(seed), t["classic"], ctypes.byref(w))
    h = t["H"]
    F = t["F"]
    blocks = np.frombuffer(w.blocks, np.uint8).reshape(9, 4096)[:F, :h * h].reshape(F, h, h).copy()
    items = np.frombuffer(w.items, np.uint8).reshape(9, 4096)[:F, :h * h].reshape(F, h, h).copy()
    chest = np.frombuffer(w.chest, np.int16).reshape(9, 6, 4)
    return {
        "blocks": blocks, "items": items, "spawn": tuple(int(x) for x in w.spawn),
        "ladder_down": np.frombuffer(w.ladder_down, np.int16).reshape(9, 2)[:F].copy(),
        "ladder_up": np.frombuffer(w.ladder_up, np.int16).reshape(9, 2)[:F].copy(),
        "chests": [[tuple(int(x) for x in chest[f, j]) for j in range(w.n_chests[f])] for f in range(F)],
        "potion": np.frombuffer(w.potion, np.uint8).copy(),
        "attempts": list(w.attempts)[:F], "potion_tie": bool(w.potion_tie),
    }


class OracleState:
    """A SimState held by the oracle (native per-env structs)."""

    def __init__(self, tier: str, n: int, max_len: int = 100_000, _handle=None, _owner=None):
        self.tier = tier
        self.n = n
        self.t = TIERS[tier]
        self._owner = _owner
        self.h = _handle if _handle is not None else lib().go_state_new(self.t["classic"], n, max_len)
        self._own = _handle is None

    def __del__(self):
        if getattr(self, "_own", False) and self.h:
            lib().go_state_free(self.h)
            self.h = None

    def _ptrs(self, arrs: dict):
        ptrs = (ctypes.c_void_p * len(FIELDS))()
        for k, name in enumerate(FIELD_NAMES):
            a = arrs.get(name)
            ptrs[k] = a.ctypes.data if a is not None else None
        return ptrs

    def import_fields(self, arrs: dict) -> None:
        shapes = field_shapes(self.tier, self.n)
        conv = {}
        for name, (dt, shape) in shapes.items():
            a = np.ascontiguousarray(np.asarray(arrs[name]).astype(dt, copy=False))
            assert a.shape == shape, (name, a.shape, shape)
            conv[name] = a
        lib().go_state_import(self.h, self._ptrs(conv))

    def export_fields(self) -> dict:
        out = alloc_fields(self.tier, self.n)
        lib().go_state_export(self.h, self._ptrs(out))
        return out

    def install_seed(self, env: int, world_seed: int, key: int) -> None:
        lib().go_state_install_seed(self.h, env, ctypes.c_uint64(world_seed), ctypes.c_uint64(key))

    def step(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.int64)
        reward = np.zeros(self.n, np.float64)
        done = np.zeros(self.n, np.bool_)
        newly = np.zeros((self.n, self.t["A"]), np.bool_)
        delta = np.zeros(self.n, np.float32)
        rc = lib().go_state_step(self.h, _ptr(a), _ptr(reward), _ptr(done), _ptr(newly), _ptr(delta))
        if rc < 0:
            bad = -1 - rc
            raise ValueError(f"invalid action id {int(a[bad])} for env {bad}")
        return reward, done, newly, delta

    def encode_symbolic(self) -> np.ndarray:
        out = np.empty((self.n, self.t["L"]), np.float32)
        lib().go_state_encode(self.h, _ptr(out))
        return out

    def render_pixels(self, px: int) -> np.ndarray:
        out = np.empty((self.n,) + pixel_shape(self.tier, px), np.uint8)
        lib().go_state_pixels(self.h, px, _ptr(out))
        return out


class OracleBatch:
    """batch.batch_reset / batch_step (batch.py:127-234) on the oracle."""

    def __init__(self, tier: str, n: int, seed: int, reset_ratio: int = 16,
                 max_episode_length: int | None = None, threads: int = 1,
                 env_offset: int = 0, n_global: int | None = None):
        self.tier = tier
        self.n = n
        self.t = TIERS[tier]
        self.h = lib().go_batch_create_shard(self.t["classic"], n, env_offset, n_global or n,
                                             ctypes.c_uint64(seed), reset_ratio,
                                             max_episode_length or 0, threads)
        self.state = OracleState(tier, n, _handle=lib().go_batch_state(self.h), _owner=self)

    # --- sharded step: the three phases of go_batch_step ----------------
    def step_a(self, actions) -> np.ndarray:
        self._a = np.ascontiguousarray(actions, dtype=np.int64)
        flags = np.zeros(2, np.int32)
        rc = lib().go_batch_step_a(self.h, _ptr(self._a), _ptr(flags))
        if rc < 0:
            bad = -1 - rc
            raise ValueError(f"invalid action {int(self._a[bad])} for env {bad}")
        return flags

    def step_b(self, flags):
        fl = np.ascontiguousarray(flags, dtype=np.int32)
        reward = np.zeros(self.n, np.float64)
        done = np.zeros(self.n, np.bool_)
        newly = np.zeros((self.n, self.t["A"]), np.bool_)
        itime = np.zeros(self.n, np.uint32)
        ifloor = np.zeros(self.n, np.uint8)
        k = lib().go_batch_step_b(self.h, _ptr(fl), _ptr(reward), _ptr(done), _ptr(newly), _ptr(itime),
                                  _ptr(ifloor))
        return reward, done, newly, {"time": itime, "floor": ifloor}, int(k)

    def step_c(self, offset: int) -> None:
        lib().go_batch_step_c(self.h, int(offset))

    def any_dark(self) -> bool:
        return bool(lib().go_state_any_dark(self.state.h))

    def encode_symbolic(self, dark: bool) -> np.ndarray:
        out = np.empty((self.n, self.t["L"]), np.float32)
        lib().go_state_encode_flag(self.state.h, 1 if dark else 0, _ptr(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().go_batch_destroy(self.h)
            self.h = None

    def step(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.int64)
        reward = np.zeros(self.n, np.float64)
        done = np.zeros(self.n, np.bool_)
        newly = np.zeros((self.n, self.t["A"]), np.bool_)
        itime = np.zeros(self.n, np.uint32)
        ifloor = np.zeros(self.n, np.uint8)
        rc = lib().go_batch_step(self.h, _ptr(a), _ptr(reward), _ptr(done), _ptr(newly),
                                 _ptr(itime), _ptr(ifloor))
        if rc < 0:
            bad = -1 - rc
            raise ValueError(f"invalid action {int(a[bad])} for env {bad}")
        return reward, done, newly, {"time": itime, "floor": ifloor}

    def episode_progress(self) -> tuple:
        """BatchState.ep_return (f64[N]) and ep_length (i64[N])."""
        ret = np.zeros(self.n, np.float64)
        length = np.zeros(self.n, np.int64)
        lib().go_batch_ep(self.h, _ptr(ret), _ptr(length))
        return ret, length

    def stats(self) -> dict:
        ep = ctypes.c_int64()
        tr = ctypes.c_double()
        ts = ctypes.c_int64()
        ach = np.zeros(self.t["A"], np.int64)
        lib().go_batch_stats(self.h, ctypes.byref(ep), ctypes.byref(tr), ctypes.byref(ts), _ptr(ach))
        return {"episodes": ep.value, "total_return": tr.value, "total_steps": ts.value,
                "ach_episodes": ach}


def random_actions(seed: int, t: int, n: int, n_actions: int, env0: int = 0) -> np.ndarray:
    """policies.RandomPolicy(seed, n_actions).actions at step t (policies.py:31-37)."""
    out = np.empty(n, np.int64)
    lib().go_random_actions(seed & 0xFFFFFFFF, t, env0, n, n_actions, _ptr(out))
    return out
