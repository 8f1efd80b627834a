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
