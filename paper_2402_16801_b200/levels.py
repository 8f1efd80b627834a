"""Level buffers for curriculum methods (UED) on the device.

The reference's level pipeline for PLR / ACCEL-style curricula
(PAPER.md:267-280): ``worldgen.make_level_params`` (worldgen.py:75-87) ->
``mutate.mutate_noise`` (mutate.py:36-44) -> ``worldgen.generate_world``
(worldgen.py:636-651) -> ``mutate.mutate_swap / mutate_rswap``
(mutate.py:58-103) -> ``state.install_world`` into an env slot
(state.py:169-249).  ``LevelBuffer`` keeps a buffer of levels (params +
generated worlds) in HBM and runs every stage on the device through the C
ABI (gr_levels_*); results equal the reference's
(tests/golden/ued_levels.npz, minted from it).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import rng
from ._lib import check, lib

OPS = {"noise": 0, "swap": 1, "rswap": 2}
NOISE_RANGE = 0.5                       # mutate.NOISE_RANGE
OCTAVE_SHAPES = ((3, 3), (9, 9), (9, 9), (9, 9))   # worldgen.OVERWORLD_OCTAVES grids, 252 angles


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _u64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64).reshape(-1))


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64).reshape(-1))


def split_angles(flat: np.ndarray) -> tuple:
    """252 flat angles -> the LevelParams.overworld_angles grids."""
    out, at = [], 0
    for shp in OCTAVE_SHAPES:
        n = shp[0] * shp[1]
        out.append(flat[at:at + n].reshape(shp))
        at += n
    return tuple(out)


class LevelBuffer:
    def __init__(self, batch, capacity: int):
        self.batch = batch
        self.capacity = int(capacity)
        self.tier = batch.tier
        self.h = ctypes.c_void_p()
        check(lib().gr_levels_create(batch.h, self.capacity, ctypes.byref(self.h)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib().gr_levels_destroy(h)
            self.h = None

    # --- params -------------------------------------------------------
    def set_params(self, first: int, seeds, angles=None, floor_seeds=None) -> None:
        """LevelParams of levels [first, first + len(seeds)); without angles /
        floor seeds they are make_level_params(seed)."""
        s = _u64(seeds)
        a = None if angles is None else np.ascontiguousarray(np.asarray(angles, np.float32).reshape(len(s), 252))
        f = None if floor_seeds is None else np.ascontiguousarray(np.asarray(floor_seeds, np.uint64).reshape(len(s), 9))
        check(lib().gr_levels_set_params(self.h, int(first), len(s), _p(s), None if a is None else _p(a),
                                         None if f is None else _p(f)))

    def params(self, first: int, count: int):
        """(seeds u64[count], angles f32[count, 252], floor_seeds u64[count, 9])."""
        s = np.zeros(count, np.uint64)
        a = np.zeros((count, 252), np.float32)
        f = np.zeros((count, 9), np.uint64)
        check(lib().gr_levels_get_params(self.h, int(first), int(count), _p(s), _p(a), _p(f)))
        return s, a, f

    # --- worlds ---------------------------------------------------------
    def generate(self, first: int, count: int) -> None:
        check(lib().gr_levels_generate(self.h, int(first), int(count)))

    def mutate(self, op: str, level_idx, streams, scale: float = NOISE_RANGE) -> None:
        """op 'noise' (params: regenerate after), 'swap' or 'rswap' (worlds, in
        place); streams: one rng.Stream (or (key, counter)) per level."""
        idx = _i64(level_idx)
        st = [s if isinstance(s, rng.Stream) else rng.Stream(*s) for s in streams]
        if len(st) != len(idx):
            raise ValueError("one stream per mutated level")
        keys = _u64([s.key for s in st])
        ctrs = _u64([s.counter for s in st])
        check(lib().gr_levels_mutate(self.h, OPS[op], len(idx), _p(idx), _p(keys), _p(ctrs), float(scale)))

    def install(self, env_idx, level_idx, keys) -> None:
        """install_world(sim, env_idx[k], level level_idx[k], keys[k])."""
        e, l, k = _i64(env_idx), _i64(level_idx), _u64(keys)
        if not (len(e) == len(l) == len(k)):
            raise ValueError("env_idx, level_idx and keys must have equal length")
        check(lib().gr_levels_install(self.h, len(e), _p(e), _p(l), _p(k)))

    def world(self, level: int) -> dict:
        """One World in the reference's layout (worldgen.World fields)."""
        from .layout import TIER_DIMS
        d = TIER_DIMS[self.tier]
        F, H, W = d["F"], d["H"], d["W"]
        out = {"blocks": np.zeros((F, H, W), np.uint8), "items": np.zeros((F, H, W), np.uint8),
               "spawn": np.zeros(2, np.int16), "ladders": np.zeros((F, 4), np.int16),
               "chests": np.zeros((F, 6, 4), np.int64), "potion": np.zeros(6, np.uint8)}
        check(lib().gr_levels_export_world(self.h, int(level), _p(out["blocks"]), _p(out["items"]), _p(out["spawn"]),
                                           _p(out["ladders"]), _p(out["chests"]), _p(out["potion"])))
        return out

    # --- interchange with the reference's level formats (serialize.py) -------
    def level_params(self, level: int):
        """serialize.LevelParams of one level."""
        from .serialize import LevelParams
        s, a, f = self.params(level, 1)
        return LevelParams(int(s[0]), a[0], f[0])

    def set_level_params(self, level: int, p) -> None:
        self.set_params(level, [p.seed], p.angles[None, :], p.floor_seeds[None, :])

    def export_world(self, level: int):
        """The level's world as serialize.World (its params included)."""
        from .serialize import World
        w = self.world(level)
        seed, tmpl = ctypes.c_uint64(), ctypes.c_uint32()
        check(lib().gr_levels_world_info(self.h, int(level), ctypes.byref(seed), ctypes.byref(tmpl)))
        return World(self.tier, w["blocks"], w["items"], w["spawn"], w["ladders"], w["chests"], w["potion"],
                     self.level_params(level), int(tmpl.value))

    def import_world(self, level: int, w) -> None:
        """Write a serialize.World (e.g. world_from_bytes of a reference blob)
        into level slot ``level``, params included; install() then places it."""
        from .layout import TIER_DIMS
        d = TIER_DIMS[self.tier]
        if w.tier != self.tier or w.blocks.shape != (d["F"], d["H"], d["W"]):
            raise ValueError(f"a {w.tier} world of shape {w.blocks.shape} does not fit a {self.tier} level buffer")
        self.set_level_params(level, w.params)
        b, it = np.ascontiguousarray(w.blocks, np.uint8), np.ascontiguousarray(w.items, np.uint8)
        sp, lad = np.ascontiguousarray(w.spawn, np.int16), np.ascontiguousarray(w.ladders, np.int16)
        ch, pot = np.ascontiguousarray(w.chests, np.int64), np.ascontiguousarray(w.potion, np.uint8)
        check(lib().gr_levels_import_world(self.h, int(level), int(w.params.seed), _p(b), _p(it), _p(sp), _p(lad),
                                           _p(ch), _p(pot), int(w.template_floors)))
