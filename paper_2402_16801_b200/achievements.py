"""Achievement names and reward weights (gridrogue.constants).

Index order is the reference's ``Achievement`` IntEnum
(/root/reference/pkg/src/gridrogue/constants.py:258-326); the classic tier
uses the first 22.  Weights are ``TierConf.ach_tier``: 1 for every classic
achievement, the Craftax tiers 1/3/5/8 for the extended ones (sums 22 and
226 = ``bench.max_return``, bench.py:36-37).  The device kernels carry the
same weights (gr_device.cuh, C_ACH_TIER).
"""

from __future__ import annotations

NAMES = (
    "COLLECT_WOOD", "PLACE_TABLE", "EAT_COW", "COLLECT_SAPLING", "COLLECT_DRINK", "MAKE_WOOD_PICKAXE",
    "MAKE_WOOD_SWORD", "PLACE_PLANT", "DEFEAT_ZOMBIE", "COLLECT_STONE", "PLACE_STONE", "EAT_PLANT",
    "DEFEAT_SKELETON", "MAKE_STONE_PICKAXE", "MAKE_STONE_SWORD", "WAKE_UP", "PLACE_FURNACE", "COLLECT_COAL",
    "COLLECT_IRON", "COLLECT_DIAMOND", "MAKE_IRON_PICKAXE", "MAKE_IRON_SWORD", "MAKE_ARROW", "MAKE_TORCH",
    "PLACE_TORCH", "MAKE_DIAMOND_SWORD", "MAKE_IRON_ARMOUR", "MAKE_DIAMOND_ARMOUR", "ENTER_GNOMISH_MINES",
    "ENTER_DUNGEON", "ENTER_SEWERS", "ENTER_VAULT", "ENTER_TROLL_MINES", "ENTER_FIRE_REALM", "ENTER_ICE_REALM",
    "ENTER_GRAVEYARD", "DEFEAT_GNOME_WARRIOR", "DEFEAT_GNOME_ARCHER", "DEFEAT_ORC_SOLDIER", "DEFEAT_ORC_MAGE",
    "DEFEAT_LIZARD", "DEFEAT_KOBOLD", "DEFEAT_TROLL", "DEFEAT_DEEP_THING", "DEFEAT_PIGMAN",
    "DEFEAT_FIRE_ELEMENTAL", "DEFEAT_FROST_TROLL", "DEFEAT_ICE_ELEMENTAL", "DAMAGE_NECROMANCER",
    "DEFEAT_NECROMANCER", "EAT_BAT", "EAT_SNAIL", "FIND_BOW", "FIRE_BOW", "COLLECT_SAPPHIRE", "LEARN_FIREBALL",
    "CAST_FIREBALL", "LEARN_ICEBALL", "CAST_ICEBALL", "COLLECT_RUBY", "MAKE_DIAMOND_PICKAXE", "OPEN_CHEST",
    "DRINK_POTION", "ENCHANT_SWORD", "ENCHANT_ARMOUR", "DEFEAT_KNIGHT", "DEFEAT_ARCHER",
)

_EXT_WEIGHTS = (1.0,) * 25 + (3.0,) * 5 + (5.0,) * 3 + (8.0,) * 3 + (3.0,) * 4 + (5.0,) * 4 + (8.0,) * 6 + \
    (3.0,) * 5 + (5.0,) * 4 + (3.0,) * 4 + (5.0,) * 4

WEIGHTS = {"classic": (1.0,) * 22, "extended": _EXT_WEIGHTS}
N_ACHIEVEMENTS = {"classic": 22, "extended": 67}


def names(tier: str) -> tuple:
    return NAMES[:N_ACHIEVEMENTS[tier]]


def max_return(tier: str) -> float:
    """bench.max_return (bench.py:36-37): the sum of the tier's weights."""
    return float(sum(WEIGHTS[tier]))
