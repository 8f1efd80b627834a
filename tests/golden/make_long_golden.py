"""Mint the north-star parity goldens from the unmodified numpy reference.

    python tests/golden/make_long_golden.py [long|north_star|pixels_px|all]

Run HERE (where /root/reference exists); the GPU box has no reference, so
the fixtures are committed and both the C oracle (tests/test_oracle_golden.py)
and the CUDA product (tests/test_gpu.py) are checked against them directly.

* ``long_<tier>_<obs>.npz`` -- BASELINE.json north star: "bit-exact ... parity
  with the CPU reference on 10^4-step random rollouts for all four variants".
  The configs of ``tests/test_gpu.py::test_long_rollout_parity_10k``:
  seed 31, ``max_episode_length`` 700, n = 32 (symbolic) / 16 classic pixels /
  12 extended pixels, BatchEnv semantics (``batch_step`` then the post-reset
  observation, ``bindings/src/gridrogue_gym/__init__.py:63-84``), actions from
  ``RandomPolicy(seed, n_actions)`` (``policies.py:22-37``).  Per step: blake2b
  digests of reward (the BatchEnv float32 cast, ``__init__.py:80``), done and
  the observation (``encode_symbolic_batch``, ``obs.py:343``, or the stacked
  per-env ``render_tiles`` frames, ``tiles.py:85``).  Every 2,500 steps: the
  full SimState digest (every field of ``state.FIELD_NAMES``, maps included)
  plus the f64 episode accumulators (``batch.py:200-201``), which pin the f64
  reward sums.
* ``long_{classic,extended}_symbolic_n1024.npz`` -- the same for 1,024 envs
  (seed 77, no episode cap: natural deaths only), the observation digested
  every 50 steps: 10^7 env-steps per tier.
* ``north_star_ext_n65536.npz`` -- the bench workload (Craftax-Symbolic,
  65,536 envs, seed 0): the reset state and observation, then 12 steps with
  reward / done / newly / info / observation / full-state digests per step
  and per-field digests at the end (maps included).
* ``pixels_px.npz`` (``python tests/golden/make_long_golden.py pixels_px``) -- every supported tile size (``tiles.SUPPORTED_TILE_PX``)
  for both tiers: 120-step BatchEnv-semantics rollouts of 8 envs (seed 5,
  ``max_episode_length`` 40) with the stacked ``render_tiles(state, px)``
  frames digested every step.

Digests: tests/_digest.py (blake2b-64 over dtype name + bytes).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
from tests._digest import digest, state_digest  # noqa: E402

LONG = {   # name: (tier, obs, n, seed, max_episode_length, observation digest every k steps)
    "classic_symbolic": ("classic", "symbolic", 32, 31, 700, 1),
    "extended_symbolic": ("extended", "symbolic", 32, 31, 700, 1),
    "classic_pixels": ("classic", "pixels", 16, 31, 700, 1),
    "extended_pixels": ("extended", "pixels", 12, 31, 700, 1),
    # 1,024 envs, natural episode ends (no cap): 10^7 env-steps per tier;
    # rewards / dones every step, observations every 50 steps
    "classic_symbolic_n1024": ("classic", "symbolic", 1024, 77, None, 50),
    "extended_symbolic_n1024": ("extended", "symbolic", 1024, 77, None, 50),
}
LONG_STEPS, LONG_EVERY = 10_000, 2500


def _ref():
    sys.path.insert(0, REF)
    import gridrogue
    return gridrogue


def long_rollout(name):
    _ref()
    from gridrogue import CLASSIC, EXTENDED
    from gridrogue.batch import BatchConfig, batch_reset, batch_step
    from gridrogue.obs import encode_symbolic_batch
    from gridrogue.policies import RandomPolicy
    from gridrogue.state import FIELD_NAMES, GameState
    from gridrogue.tiles import render_tiles

    tier, obs_mode, n, seed, max_len, obs_every = LONG[name]
    t = {"classic": CLASSIC, "extended": EXTENDED}[tier]
    px = 7 if tier == "classic" else 10
    bs = batch_reset(BatchConfig(n_envs=n, tier=t, max_episode_length=max_len), seed)
    pol = RandomPolicy(seed, t.n_actions)

    def observe():
        if obs_mode == "symbolic":
            return encode_symbolic_batch(bs.sim)
        return np.stack([render_tiles(GameState(bs.sim.view(slice(i, i + 1))), px) for i in range(n)])

    def full_state():
        return state_digest({f: getattr(bs.sim, f) for f in FIELD_NAMES}, FIELD_NAMES)

    reset = np.array([full_state(), digest(observe())], np.uint64)
    rew, done, obs, ckpt = [], [], [], []
    t0 = time.time()
    for k in range(LONG_STEPS):
        bs, out = batch_step(bs, pol.actions(bs.sim))
        rew.append(digest(out.reward.astype(np.float32)))
        done.append(digest(out.done))
        obs.append(digest(observe()) if k % obs_every == 0 else 0)
        if (k + 1) % LONG_EVERY == 0:
            ckpt.append([full_state(), digest(bs.ep_return, bs.ep_length)])
            print(f"  {name}: step {k + 1} ({time.time() - t0:.0f} s)", flush=True)
    st = bs.stats
    np.savez_compressed(
        os.path.join(OUT, f"long_{name}.npz"), tier=tier, obs_mode=obs_mode, n=n, steps=LONG_STEPS,
        seed=seed, max_len=max_len or 0, every=LONG_EVERY, tile_px=px, obs_every=obs_every, reset=reset,
        reward=np.array(rew, np.uint64), done=np.array(done, np.uint64), obs=np.array(obs, np.uint64),
        ckpt=np.array(ckpt, np.uint64),
        final_fields=np.array([digest(getattr(bs.sim, f)) for f in FIELD_NAMES], np.uint64),
        episodes=np.int64(st.episodes), total_steps=np.int64(st.total_steps),
        ach_episodes=np.asarray(st.ach_episodes, np.int64), level_seeds=bs.level_seeds())


NS_N, NS_SEED, NS_STEPS = 65536, 0, 12


def north_star():
    _ref()
    from gridrogue import EXTENDED
    from gridrogue.batch import BatchConfig, batch_reset, batch_step
    from gridrogue.obs import encode_symbolic_batch
    from gridrogue.policies import RandomPolicy
    from gridrogue.state import FIELD_NAMES

    t0 = time.time()
    bs = batch_reset(BatchConfig(n_envs=NS_N, tier=EXTENDED), NS_SEED)
    print(f"  north_star: reset {time.time() - t0:.0f} s", flush=True)
    pol = RandomPolicy(NS_SEED, EXTENDED.n_actions)

    def full_state():
        return state_digest({f: getattr(bs.sim, f) for f in FIELD_NAMES}, FIELD_NAMES)

    reset = np.array([full_state(), digest(encode_symbolic_batch(bs.sim))], np.uint64)
    rec = {k: [] for k in ("reward", "done", "newly", "info", "obs", "state")}
    for k in range(NS_STEPS):
        bs, out = batch_step(bs, pol.actions(bs.sim))
        rec["reward"].append(digest(out.reward.astype(np.float32)))
        rec["done"].append(digest(out.done))
        rec["newly"].append(digest(out.newly))
        rec["info"].append(digest(out.info["time"], out.info["floor"]))
        rec["obs"].append(digest(encode_symbolic_batch(bs.sim)))
        rec["state"].append(full_state())
        print(f"  north_star: step {k + 1} ({time.time() - t0:.0f} s, {int(out.done.sum())} done)", flush=True)
    st = bs.stats
    np.savez_compressed(
        os.path.join(OUT, f"north_star_ext_n{NS_N}.npz"), tier="extended", n=NS_N, steps=NS_STEPS,
        seed=NS_SEED, reset=reset, **{k: np.array(v, np.uint64) for k, v in rec.items()},
        final_fields=np.array([digest(getattr(bs.sim, f)) for f in FIELD_NAMES], np.uint64),
        episode_acc=np.uint64(digest(bs.ep_return, bs.ep_length)),
        episodes=np.int64(st.episodes), level_seeds_digest=np.uint64(digest(bs.level_seeds())))


def pixels_px():
    _ref()
    from gridrogue import CLASSIC, EXTENDED
    from gridrogue.batch import BatchConfig, batch_reset, batch_step
    from gridrogue.policies import RandomPolicy
    from gridrogue.state import GameState
    from gridrogue.tiles import render_tiles, SUPPORTED_TILE_PX
    out = {"px": np.array(SUPPORTED_TILE_PX, np.int64)}
    n, steps, seed, ml = 8, 120, 5, 40
    for tier, t in (("classic", CLASSIC), ("extended", EXTENDED)):
        for px in SUPPORTED_TILE_PX:
            bs = batch_reset(BatchConfig(n_envs=n, tier=t, max_episode_length=ml), seed)
            pol = RandomPolicy(seed, t.n_actions)
            frames = lambda: np.stack([render_tiles(GameState(bs.sim.view(slice(i, i + 1))), px) for i in range(n)])
            dg = [digest(frames())]
            for k in range(steps):
                bs, _ = batch_step(bs, pol.actions(bs.sim))
                dg.append(digest(frames()))
            out[f"{tier}_{px}"] = np.array(dg, np.uint64)
    np.savez_compressed(os.path.join(OUT, "pixels_px.npz"), n=n, steps=steps, seed=seed, max_len=ml, **out)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "pixels_px":
        pixels_px()
    if what in ("long", "all"):
        for nm in (sys.argv[2:] or LONG):
            long_rollout(nm)
    if what in ("north_star", "all"):
        north_star()
    print("written to", OUT)
