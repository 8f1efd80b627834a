"""SimState field layout of the reference (state._SHAPES, state.py:29-125).

(name, dtype, trailing shape) per field, in ``FIELD_NAMES`` order; F/H/W/A
are the tier's floors, map height/width and achievement count, the numbers
are the fixed lane capacities (constants.py:502-508).  The C ABI's state
channel (gr_export_field / gr_import_field) moves exactly these arrays.
"""

from __future__ import annotations

import numpy as np

from ._lib import FIELD_NAMES

_LAYOUT = (
    ("blocks", np.uint8, ("F", "H", "W")), ("items", np.uint8, ("F", "H", "W")),
    ("ladder_down", np.int16, ("F", 2)), ("ladder_up", np.int16, ("F", 2)),
    ("spawn0", np.int16, (2,)), ("potion_map", np.uint8, (6,)),
    ("chest_pos", np.int16, ("F", 6, 2)), ("chest_loot", np.uint8, ("F", 6)),
    ("chest_qty", np.uint8, ("F", 6)), ("chest_aux", np.uint8, ("F", 6)),
    ("necro_pos", np.int16, (2,)), ("params_seed", np.uint64, ()),
    ("pfloor", np.uint8, ()), ("prow", np.int16, ()), ("pcol", np.int16, ()),
    ("facing", np.uint8, ()), ("health", np.float32, ()), ("food", np.float32, ()),
    ("drink", np.float32, ()), ("energy", np.float32, ()), ("mana", np.float32, ()),
    ("xp", np.uint8, ()), ("dex", np.uint8, ()), ("str_", np.uint8, ()), ("intel", np.uint8, ()),
    ("sword_tier", np.uint8, ()), ("pick_tier", np.uint8, ()), ("has_bow", np.bool_, ()),
    ("sword_ench", np.uint8, ()), ("bow_ench", np.uint8, ()), ("armour", np.uint8, (4,)),
    ("armour_ench", np.uint8, (4,)), ("learned_fire", np.bool_, ()), ("learned_ice", np.bool_, ()),
    ("sleeping", np.bool_, ()), ("resting", np.bool_, ()),
    ("inv_wood", np.uint8, ()), ("inv_stone", np.uint8, ()), ("inv_coal", np.uint8, ()),
    ("inv_iron", np.uint8, ()), ("inv_diamond", np.uint8, ()), ("inv_sapphire", np.uint8, ()),
    ("inv_ruby", np.uint8, ()), ("inv_sapling", np.uint8, ()), ("inv_torch", np.uint8, ()),
    ("inv_arrow", np.uint8, ()), ("inv_book", np.uint8, ()), ("inv_potion", np.uint8, (6,)),
    ("mel_pos", np.int16, ("F", 3, 2)), ("mel_hp", np.float32, ("F", 3)), ("mel_cd", np.uint8, ("F", 3)),
    ("mel_alive", np.bool_, ("F", 3)), ("mel_type", np.uint8, ("F", 3)),
    ("ran_pos", np.int16, ("F", 2, 2)), ("ran_hp", np.float32, ("F", 2)), ("ran_cd", np.uint8, ("F", 2)),
    ("ran_alive", np.bool_, ("F", 2)), ("ran_type", np.uint8, ("F", 2)),
    ("pas_pos", np.int16, ("F", 3, 2)), ("pas_hp", np.float32, ("F", 3)),
    ("pas_alive", np.bool_, ("F", 3)), ("pas_type", np.uint8, ("F", 3)),
    ("pproj_pos", np.int16, (3, 2)), ("pproj_dir", np.uint8, (3,)), ("pproj_type", np.uint8, (3,)),
    ("pproj_ttl", np.uint8, (3,)), ("pproj_alive", np.bool_, (3,)), ("pproj_dmg", np.float32, (3, 3)),
    ("eproj_pos", np.int16, (3, 2)), ("eproj_dir", np.uint8, (3,)), ("eproj_type", np.uint8, (3,)),
    ("eproj_ttl", np.uint8, (3,)), ("eproj_alive", np.bool_, (3,)), ("eproj_dmg", np.float32, (3, 3)),
    ("plant_pos", np.int16, (10, 2)), ("plant_age", np.uint16, (10,)), ("plant_alive", np.bool_, (10,)),
    ("ach", np.bool_, ("A",)), ("time", np.uint32, ()), ("rng_key", np.uint64, ()),
    ("floors_visited", np.bool_, ("F",)), ("floor_cleared", np.bool_, ("F",)),
    ("boss_hp", np.float32, ()), ("boss_wave", np.uint8, ()), ("boss_vuln", np.bool_, ()),
    ("boss_timer", np.uint8, ()), ("clocks", np.uint16, (6,)), ("done", np.bool_, ()),
)
assert tuple(n for n, _, _ in _LAYOUT) == FIELD_NAMES

TIER_DIMS = {"classic": {"F": 1, "H": 64, "W": 64, "A": 22}, "extended": {"F": 9, "H": 48, "W": 48, "A": 67}}


def field_shapes(tier: str, n: int) -> dict:
    """{name: (dtype, full shape)} of a SimState of n envs."""
    d = TIER_DIMS[tier]
    return {name: (np.dtype(dt), (n,) + tuple(d[x] if isinstance(x, str) else x for x in shp))
            for name, dt, shp in _LAYOUT}
