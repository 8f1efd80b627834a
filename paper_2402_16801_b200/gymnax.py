"""gymnax-style facade over the batched environment.

Craftax's public entry points are ``make_craftax_env_from_name(name,
auto_reset)``, ``env.reset(key, params)`` and ``env.step(key, state, action,
params)`` batched over a leading env axis.  The reference mirrors the
reset/step shape through gridrogue_gym.BatchEnv; variant
names map to (tier, observation) as in SURVEY.md section 0.

Step randomness lives in per-env state (rng_key + time, _kern.py:38-46), so
``step`` ignores its ``key``; ``reset`` uses its key as the batch_reset seed.
The returned ``state`` is an opaque handle to device-resident SoA state.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .env import GridrogueBatch, TIERS, pixel_shape, DEFAULT_TILE_PX

VARIANTS = {
    "Craftax-Classic-Symbolic": ("classic", "symbolic"),
    "Craftax-Classic-Pixels": ("classic", "pixels"),
    "Craftax-Symbolic": ("extended", "symbolic"),
    "Craftax-Pixels": ("extended", "pixels"),
}


@dataclass(frozen=True)
class EnvParams:
    n_envs: int = 1024
    max_episode_length: int | None = None
    reset_ratio: int = 16
    device: int = 0
    tile_px: int | None = None


@dataclass
class EnvState:
    """Opaque handle: the batch lives on the device and is updated in place."""
    batch: GridrogueBatch
    step_count: int = 0


class _Discrete:
    def __init__(self, n):
        self.n = n
        self.shape = ()


class _Box:
    def __init__(self, shape, dtype):
        self.shape = shape
        self.dtype = dtype


def _seed_of(key) -> int:
    if key is None:
        return 0
    arr = np.asarray(key).astype(np.uint64).ravel()
    seed = 0
    for v in arr:
        seed = (seed * 0x9E3779B97F4A7C15 + int(v)) & 0xFFFFFFFFFFFFFFFF
    return seed


class CraftaxEnv:
    def __init__(self, name: str, tier: str, obs_mode: str, auto_reset: bool = True):
        if not auto_reset:
            raise ValueError("only auto-resetting environments exist on this path (batch.py:193-234)")
        self.name = name
        self.tier = tier
        self.obs_mode = obs_mode

    @property
    def default_params(self) -> EnvParams:
        return EnvParams()

    def num_actions(self, params: EnvParams | None = None) -> int:
        return TIERS[self.tier]["n_actions"]

    def action_space(self, params: EnvParams | None = None):
        return _Discrete(self.num_actions(params))

    def observation_space(self, params: EnvParams | None = None):
        p = params or self.default_params
        if self.obs_mode == "symbolic":
            return _Box((TIERS[self.tier]["obs"],), np.float32)
        return _Box(pixel_shape(self.tier, p.tile_px or DEFAULT_TILE_PX[self.tier]), np.uint8)

    def reset(self, key, params: EnvParams | None = None):
        p = params or self.default_params
        batch = GridrogueBatch(p.n_envs, self.tier, _seed_of(key), self.obs_mode,
                               p.max_episode_length, p.tile_px, p.device, p.reset_ratio)
        obs = batch.reset()
        return obs, EnvState(batch)

    def step(self, key, state: EnvState, action, params: EnvParams | None = None):
        obs, reward, done, newly, time, floor = state.batch.step(action)
        state.step_count += 1
        info = {"time": time, "floor": floor, "newly_unlocked": newly}
        return obs, state, reward, done.bool(), info


def make_craftax_env_from_name(name: str, auto_reset: bool = True) -> CraftaxEnv:
    base = name[:-3] if name.endswith("-v1") else name
    if base not in VARIANTS:
        raise ValueError(f"unknown environment {name!r}; expected one of {sorted(VARIANTS)}")
    tier, obs = VARIANTS[base]
    return CraftaxEnv(name, tier, obs, auto_reset)
