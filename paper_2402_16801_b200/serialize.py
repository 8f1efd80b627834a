"""Versioned serialization of device batches (gridrogue.serialize).

The reference's episode-state format (serialize.py:155-194): a zip of npy
arrays (``numpy.savez``) with a ``__meta__`` JSON entry
``{"format": "game_state", "version": 1, "tier": ...}``, one array per
SimState field in ``FIELD_NAMES`` order and layout, plus
``max_episode_length``; the JSON debug form mirrors it with plain lists.
``state_to_bytes`` / ``state_from_bytes`` here read and write exactly that
format from / into a device batch, so blobs move freely between the
reference and this library (tests: tests/test_serialize_cpu.py against the
reference's own reader and writer, tests/test_gpu.py round trips on the
device).

The reference's level formats (serialize.py:43-151) move UED levels between
the reference and ``levels.LevelBuffer``: ``params_*`` (format
``"level_params"``: seed, nine floor seeds, the four overworld angle grids)
and ``world_*`` (format ``"world"``: per floor blocks / items / ambient light
/ spawn / ladders / chests, the potion permutation and the nested params
blob).  ``LevelBuffer.export_world`` / ``import_world`` convert a device level
slot to / from ``World``; ``world_to_bytes`` writes the bytes the reference
writes for the same world, and ``world_from_bytes`` reads its blobs.

``batch_to_bytes`` / ``batch_from_bytes`` extend it to a whole
``BatchState`` checkpoint (format ``"batch_state"``, this library's
extension): the SimState arrays plus the running episode returns and
lengths, ``EpisodeStats``, the step counter that keys the reset pool, and
the batch configuration (seed, reset ratio, global size, shard offset).
Resuming from one continues the run bit for bit.
"""

from __future__ import annotations

import io
import json
from dataclasses import dataclass, field

import numpy as np

from ._lib import FIELD_NAMES
from .layout import field_shapes

FORMAT_VERSION = 1
DEFAULT_MAX_EPISODE_LENGTH = 100_000   # TierConf.max_episode_length (constants.py:527-545)


def _pack(kind: str, tier: str, arrays: dict, extra_meta: dict | None = None) -> bytes:
    meta = {"format": kind, "version": FORMAT_VERSION, "tier": tier}
    if extra_meta:
        meta.update(extra_meta)
    buf = io.BytesIO()
    np.savez(buf, __meta__=np.frombuffer(json.dumps(meta).encode(), np.uint8), **arrays)
    return buf.getvalue()


def _unpack(blob: bytes, kind: str):
    data = np.load(io.BytesIO(blob), allow_pickle=False)
    meta = json.loads(bytes(data["__meta__"]).decode())
    if meta.get("format") != kind:
        raise ValueError(f"expected a {kind} blob, got {meta.get('format')!r}")
    if meta.get("version") != FORMAT_VERSION:
        raise ValueError(f"unsupported {kind} version {meta.get('version')!r}")
    return meta, data


def _max_len(gb) -> int:
    return int(gb.cfg.max_episode_length) or DEFAULT_MAX_EPISODE_LENGTH


def _fields_of(data, tier: str) -> dict:
    n = int(data["pfloor"].shape[0])
    shapes = field_shapes(tier, n)
    out = {}
    for name in FIELD_NAMES:
        a = np.ascontiguousarray(data[name])
        dt, shape = shapes[name]
        if a.dtype != dt or a.shape != shape:
            raise ValueError(f"field {name}: expected {dt}{shape}, got {a.dtype}{a.shape}")
        out[name] = a
    return out


def _new_batch(tier: str, n: int, max_len: int, **kw):
    # no reset: the imported state replaces the whole SimState (gr_import_field
    # marks the handle ready to step); gb.observe() renders it
    from .env import GridrogueBatch
    return GridrogueBatch(n, tier, kw.pop("seed", 0), kw.pop("obs_mode", "symbolic"),
                          max_episode_length=None if max_len == DEFAULT_MAX_EPISODE_LENGTH else max_len, **kw)


# --- game_state: the reference format ------------------------------------------

def state_to_bytes(gb) -> bytes:
    """serialize.state_to_bytes (serialize.py:155-159) of the batch's SimState."""
    arrays = gb.export_state()
    arrays["max_episode_length"] = np.int64(_max_len(gb))
    return _pack("game_state", gb.tier, arrays)


def load_state(gb, blob: bytes) -> None:
    """Overwrite the batch's SimState with a game_state blob of the same size and tier."""
    meta, data = _unpack(blob, "game_state")
    if meta["tier"] != gb.tier:
        raise ValueError(f"blob tier {meta['tier']!r} != batch tier {gb.tier!r}")
    if int(data["max_episode_length"]) != _max_len(gb):
        raise ValueError("blob max_episode_length differs from the batch's")
    fields = _fields_of(data, gb.tier)
    if fields["pfloor"].shape[0] != gb.n:
        raise ValueError(f"blob has {fields['pfloor'].shape[0]} envs, the batch {gb.n}")
    gb.import_state(fields)


def state_from_bytes(blob: bytes, **batch_kwargs):
    """serialize.state_from_bytes (serialize.py:162-173) into a new device batch."""
    meta, data = _unpack(blob, "game_state")
    fields = _fields_of(data, meta["tier"])
    gb = _new_batch(meta["tier"], fields["pfloor"].shape[0], int(data["max_episode_length"]), **batch_kwargs)
    gb.import_state(fields)
    return gb


def state_to_json(gb) -> dict:
    """serialize.state_to_json (serialize.py:176-183)."""
    doc = {"format": "game_state", "version": FORMAT_VERSION, "tier": gb.tier,
           "max_episode_length": _max_len(gb)}
    for name, a in gb.export_state().items():
        doc[name] = a.tolist()
    return doc


def state_from_json(doc: dict, **batch_kwargs):
    """serialize.state_from_json (serialize.py:186-194) into a new device batch."""
    if doc.get("format") != "game_state" or doc.get("version") != FORMAT_VERSION:
        raise ValueError("not a game_state v1 document")
    tier = doc["tier"]
    n = len(doc["pfloor"])
    shapes = field_shapes(tier, n)
    fields = {name: np.array(doc[name], shapes[name][0]).reshape(shapes[name][1]) for name in FIELD_NAMES}
    gb = _new_batch(tier, n, int(doc["max_episode_length"]), **batch_kwargs)
    gb.import_state(fields)
    return gb


# --- level_params (serialize.py:43-74) ---------------------------------------------

OCTAVE_SHAPES = ((3, 3), (9, 9), (9, 9), (9, 9))   # worldgen.OVERWORLD_OCTAVES grids (worldgen.py:29,69)
# constants.FLOOR_AMBIENT (constants.py:386): FloorMap.light_base is this constant per floor
FLOOR_AMBIENT = (1.0, 1.0, 0.0, 1.0, 1.0, 0.0, 1.0, 0.0, 0.0)


@dataclass
class LevelParams:
    """worldgen.LevelParams (worldgen.py:57-66): angles flat (252 float32, the
    four grids in order), nine per-floor seeds."""
    seed: int
    angles: np.ndarray
    floor_seeds: np.ndarray

    def __post_init__(self):
        self.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        self.angles = np.ascontiguousarray(np.asarray(self.angles, np.float32).reshape(252))
        self.floor_seeds = np.ascontiguousarray(np.asarray(self.floor_seeds, np.uint64).reshape(9))

    @property
    def overworld_angles(self) -> tuple:
        out, at = [], 0
        for shp in OCTAVE_SHAPES:
            out.append(self.angles[at:at + shp[0] * shp[1]].reshape(shp))
            at += shp[0] * shp[1]
        return tuple(out)


def params_to_bytes(p: LevelParams) -> bytes:
    arrays = {"seed": np.uint64(p.seed), "per_floor_seeds": p.floor_seeds.copy()}
    for i, grid in enumerate(p.overworld_angles):
        arrays[f"angles_{i}"] = grid
    return _pack("level_params", "", arrays)


def params_from_bytes(blob: bytes) -> LevelParams:
    _, data = _unpack(blob, "level_params")
    angles = np.concatenate([np.asarray(data[f"angles_{i}"], np.float32).reshape(-1)
                             for i in range(len(OCTAVE_SHAPES))])
    return LevelParams(int(data["seed"]), angles, np.asarray(data["per_floor_seeds"], np.uint64))


def params_to_json(p: LevelParams) -> dict:
    return {"format": "level_params", "version": FORMAT_VERSION, "seed": int(p.seed),
            "per_floor_seeds": [int(x) for x in p.floor_seeds],
            "overworld_angles": [g.tolist() for g in p.overworld_angles]}


def params_from_json(doc: dict) -> LevelParams:
    angles = np.concatenate([np.array(g, np.float32).reshape(-1) for g in doc["overworld_angles"]])
    return LevelParams(int(doc["seed"]), angles, np.array([int(x) for x in doc["per_floor_seeds"]], np.uint64))


# --- world (serialize.py:77-151) -----------------------------------------------------

@dataclass
class World:
    """worldgen.World in LevelBuffer layout: blocks / items [F, H, W] u8,
    spawn (floor 0) [2], ladders [F, 4] (down r, c, up r, c; -1 none), chests
    [F, 6, 4] (r, c, loot, qty; rows of -1 pad), potion [6]; template_floors:
    bit f set when floor f is the _template_floor fallback (its spawn is the
    map centre; other lower floors spawn on their up ladder)."""
    tier: str
    blocks: np.ndarray
    items: np.ndarray
    spawn: np.ndarray
    ladders: np.ndarray
    chests: np.ndarray
    potion: np.ndarray
    params: LevelParams
    template_floors: int = 0

    def floor_spawn(self, f: int) -> tuple:
        if f == 0:
            return (int(self.spawn[0]), int(self.spawn[1]))
        if (self.template_floors >> f) & 1:
            return (self.blocks.shape[1] // 2, self.blocks.shape[2] // 2)
        return (int(self.ladders[f, 2]), int(self.ladders[f, 3]))

    def floor_chests(self, f: int) -> list:
        return [tuple(int(v) for v in row) for row in self.chests[f] if row[0] >= 0]


def world_to_bytes(w: World) -> bytes:
    arrays = {"potion_permutation": np.asarray(w.potion, np.uint8), "n_floors": np.int64(len(w.blocks))}
    for f in range(len(w.blocks)):
        arrays[f"floor{f}_blocks"] = np.ascontiguousarray(w.blocks[f])
        arrays[f"floor{f}_items"] = np.ascontiguousarray(w.items[f])
        arrays[f"floor{f}_light"] = np.full(w.blocks[f].shape, FLOOR_AMBIENT[f], np.float32)
        arrays[f"floor{f}_spawn"] = np.array(w.floor_spawn(f), np.int16)
        arrays[f"floor{f}_ladder_down"] = np.array(w.ladders[f, 0:2], np.int16)
        arrays[f"floor{f}_ladder_up"] = np.array(w.ladders[f, 2:4], np.int16)
        ch = w.floor_chests(f)
        arrays[f"floor{f}_chests"] = np.array(ch, np.int64) if ch else np.zeros((0, 4), np.int64)
    arrays["params"] = np.frombuffer(params_to_bytes(w.params), np.uint8)
    return _pack("world", w.tier, arrays)


def _world_of(tier, floors, potion, chests, params) -> World:
    F = len(floors)
    H, W = floors[0]["blocks"].shape
    lad = np.full((F, 4), -1, np.int16)
    ch = np.full((F, 6, 4), -1, np.int64)
    tmpl = 0
    for f, fd in enumerate(floors):
        if fd["ladder_down"] is not None:
            lad[f, 0:2] = fd["ladder_down"]
        if fd["ladder_up"] is not None:
            lad[f, 2:4] = fd["ladder_up"]
        if f > 0 and tuple(fd["spawn"]) != tuple(lad[f, 2:4]):
            tmpl |= 1 << f      # the template floor's centre spawn (worldgen.py:565-566)
        for j, row in enumerate(chests[f]):
            ch[f, j] = row
    return World(tier, np.stack([fd["blocks"] for fd in floors]).astype(np.uint8),
                 np.stack([fd["items"] for fd in floors]).astype(np.uint8),
                 np.array(floors[0]["spawn"], np.int16), lad, ch, np.asarray(potion, np.uint8), params, tmpl)


def world_from_bytes(blob: bytes) -> World:
    meta, data = _unpack(blob, "world")
    floors, chests = [], []
    for f in range(int(data["n_floors"])):
        ld = tuple(int(x) for x in data[f"floor{f}_ladder_down"])
        lu = tuple(int(x) for x in data[f"floor{f}_ladder_up"])
        floors.append({"blocks": data[f"floor{f}_blocks"], "items": data[f"floor{f}_items"],
                       "spawn": tuple(int(x) for x in data[f"floor{f}_spawn"]),
                       "ladder_down": None if ld == (-1, -1) else ld, "ladder_up": None if lu == (-1, -1) else lu})
        chests.append([tuple(int(v) for v in row) for row in data[f"floor{f}_chests"]])
    return _world_of(meta["tier"], floors, data["potion_permutation"], chests,
                     params_from_bytes(bytes(data["params"])))


def world_to_json(w: World) -> dict:
    F = len(w.blocks)
    return {"format": "world", "version": FORMAT_VERSION, "tier": w.tier,
            "potion_permutation": np.asarray(w.potion).tolist(),
            "chests": [[list(c) for c in w.floor_chests(f)] for f in range(F)],
            "floors": [{"blocks": w.blocks[f].tolist(), "items": w.items[f].tolist(),
                        "ambient_light": float(np.float32(FLOOR_AMBIENT[f])),
                        "spawn": list(w.floor_spawn(f)),
                        "ladder_down": [int(x) for x in w.ladders[f, 0:2]] if w.ladders[f, 0] >= 0 else None,
                        "ladder_up": [int(x) for x in w.ladders[f, 2:4]] if w.ladders[f, 2] >= 0 else None}
                       for f in range(F)],
            "params": params_to_json(w.params)}


def world_from_json(doc: dict) -> World:
    if doc.get("format") != "world" or doc.get("version") != FORMAT_VERSION:
        raise ValueError("not a world v1 document")
    floors = [{"blocks": np.array(fd["blocks"], np.uint8), "items": np.array(fd["items"], np.uint8),
               "spawn": tuple(fd["spawn"]),
               "ladder_down": tuple(fd["ladder_down"]) if fd["ladder_down"] else None,
               "ladder_up": tuple(fd["ladder_up"]) if fd["ladder_up"] else None} for fd in doc["floors"]]
    return _world_of(doc["tier"], floors, doc["potion_permutation"], [[tuple(c) for c in lanes]
                                                                      for lanes in doc["chests"]],
                     params_from_json(doc["params"]))


# --- batch_state: checkpoint / resume (this library's extension) ----------------

def batch_to_bytes(gb) -> bytes:
    arrays = gb.export_state()
    arrays["max_episode_length"] = np.int64(_max_len(gb))
    ep_return, ep_length = gb.episode_progress()
    st = gb.stats()
    arrays.update(ep_return=ep_return, ep_length=ep_length, step_index=np.int64(gb.step_index),
                  stats_episodes=np.int64(st["episodes"]), stats_total_steps=np.int64(st["total_steps"]),
                  stats_total_return=np.float64(st["total_return"]), stats_ach_episodes=st["ach_episodes"])
    cfg = {"seed": int(gb.cfg.seed), "reset_ratio": int(gb.cfg.reset_ratio),
           "n_envs_global": int(gb.cfg.n_envs_global), "env_offset": int(gb.cfg.env_offset)}
    return _pack("batch_state", gb.tier, arrays, {"batch": cfg})


def batch_from_bytes(blob: bytes, **batch_kwargs):
    """A device batch that continues the checkpointed run exactly."""
    meta, data = _unpack(blob, "batch_state")
    fields = _fields_of(data, meta["tier"])
    cfg = meta["batch"]
    n = fields["pfloor"].shape[0]
    gb = _new_batch(meta["tier"], n, int(data["max_episode_length"]), seed=cfg["seed"],
                    reset_ratio=cfg["reset_ratio"], n_envs_global=cfg["n_envs_global"],
                    env_offset=cfg["env_offset"], **batch_kwargs)
    gb.import_state(fields)
    gb.set_episode_progress(data["ep_return"], data["ep_length"])
    gb.set_stats({"episodes": int(data["stats_episodes"]), "total_steps": int(data["stats_total_steps"]),
                  "total_return": float(data["stats_total_return"]),
                  "ach_episodes": np.asarray(data["stats_ach_episodes"])})
    gb.step_index = int(data["step_index"])
    return gb
