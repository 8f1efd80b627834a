"""Mint golden vectors from the reference (run HERE, where /root/reference exists).

    python tests/golden/make_golden.py

Imports the unmodified numpy reference read-only from
/root/reference/pkg/src (gridrogue) and writes small fixtures next to this
script.  The fixtures pin the C oracle (tests/test_oracle_golden.py), which in
turn is the checker for the CUDA product on the GPU box, where the reference
does not exist.  Everything is digested with blake2b-64 (see ``digest``) so
the fixtures stay small; the scrambled start states of the fuzz goldens are
stored in full (npz, compressed).

Hazard H1/H5 of SURVEY.md: numpy's float32 sin/cos and argsort are
host-SIMD-dependent, so ``meta.json`` records numpy's version and SIMD
features for the run that produced these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays) -> int:
    h = hashlib.blake2b(digest_size=8)
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return int.from_bytes(h.digest(), "little")


def state_digest(fields: dict, names) -> int:
    return digest(*[fields[n] for n in names])


def main() -> None:
    sys.path.insert(0, REF)
    from gridrogue import CLASSIC, EXTENDED, make_level_params, generate_world
    from gridrogue import rng as R
    from gridrogue.batch import BatchConfig, batch_reset, batch_step
    from gridrogue.engine import step_batch, reset, step
    from gridrogue._kern import Workspace
    from gridrogue.obs import encode_symbolic_batch
    from gridrogue.policies import RandomPolicy
    from gridrogue.state import FIELD_NAMES, GameState
    from gridrogue.tiles import render_tiles

    sys.path.insert(0, OUT)
    from scramble import scramble

    tiers = {"classic": CLASSIC, "extended": EXTENDED}

    # ---- rng known answers (rng.py)
    keys = np.array([0, 1, 42, 2**63 + 5, 0xDEADBEEFCAFEBABE], np.uint64)
    ctrs = np.arange(0, 50, dtype=np.uint64)
    h2 = np.array([[R.hash2(int(k), int(c)) for c in ctrs] for k in keys], np.uint64)
    v32 = R.vuniform32(np.uint32(0x1234567), np.arange(4096, dtype=np.uint32))
    xs = (np.arange(200_000, dtype=np.float64) * (2 * np.pi / 200_000)).astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), keys=keys, ctrs=ctrs, hash2=h2, vuniform32=v32,
                        trig_x=xs[::97], sin=np.sin(xs)[::97], cos=np.cos(xs)[::97],
                        trig_digest=np.array([digest(np.sin(xs)), digest(np.cos(xs))], np.uint64))

    # ---- worlds: digests of make_level_params(seed) -> generate_world
    worlds = {}
    for name, n_seeds in (("classic", 400), ("extended", 120)):
        t = tiers[name]
        rows = []
        for seed in range(n_seeds):
            w = generate_world(make_level_params(seed), t)
            parts = []
            for fm in w.floors:
                parts += [fm.blocks, fm.items, np.array(fm.spawn, np.int64),
                          np.array(fm.ladder_down or (-1, -1), np.int64),
                          np.array(fm.ladder_up or (-1, -1), np.int64)]
            ch = np.array([c for lanes in w.chests for c in lanes] or np.zeros((0, 4)), np.int64)
            rows.append([digest(*parts), digest(ch.reshape(-1, 4)), digest(w.potion_permutation.astype(np.int64))])
        worlds[name] = np.array(rows, np.uint64)
    np.savez_compressed(os.path.join(OUT, "worlds.npz"), **worlds)

    # ---- batched rollouts under BatchEnv semantics (batch_step + post-reset obs)
    def rollout(tier_name, n, steps, seed, max_len=None, obs=True, pix_every=0):
        t = tiers[tier_name]
        bs = batch_reset(BatchConfig(n_envs=n, tier=t, max_episode_length=max_len), seed)
        pol = RandomPolicy(seed, t.n_actions)
        rec = {k: [] for k in ("state", "reward", "done", "newly", "info", "obs", "pix")}
        sim0 = {f: getattr(bs.sim, f) for f in FIELD_NAMES}
        rec_reset = [state_digest(sim0, FIELD_NAMES), digest(encode_symbolic_batch(bs.sim))]
        px = 7 if tier_name == "classic" else 10
        for k in range(steps):
            a = pol.actions(bs.sim)
            bs, out = batch_step(bs, a)
            rec["state"].append(state_digest({f: getattr(bs.sim, f) for f in FIELD_NAMES}, FIELD_NAMES))
            rec["reward"].append(digest(out.reward))
            rec["done"].append(digest(out.done))
            rec["newly"].append(digest(out.newly))
            rec["info"].append(digest(out.info["time"], out.info["floor"]))
            rec["obs"].append(digest(encode_symbolic_batch(bs.sim)) if obs else 0)
            if pix_every and k % pix_every == 0:
                frames = np.stack([render_tiles(GameState(bs.sim.view(slice(i, i + 1))), px)
                                   for i in range(n)])
                rec["pix"].append(digest(frames))
            else:
                rec["pix"].append(0)
        final = np.array([digest(getattr(bs.sim, f)) for f in FIELD_NAMES], np.uint64)
        st = bs.stats
        return dict(reset=np.array(rec_reset, np.uint64),
                    **{k: np.array(v, np.uint64) for k, v in rec.items()},
                    final_fields=final, episodes=np.int64(st.episodes),
                    total_steps=np.int64(st.total_steps),
                    ach_episodes=np.asarray(st.ach_episodes if st.ach_episodes is not None
                                            else np.zeros(t.n_achievements), np.int64),
                    level_seeds=bs.level_seeds())

    cfgs = {
        "classic_n64_s0": ("classic", 64, 600, 0, None, 20),
        "extended_n64_s0": ("extended", 64, 500, 0, None, 25),
        "classic_n48_s3": ("classic", 48, 300, 3, None, 0),
        "extended_n40_s5": ("extended", 40, 300, 5, None, 0),
        "extended_stress_n32_L16": ("extended", 32, 120, 1, 16, 10),
        "classic_stress_n32_L16": ("classic", 32, 120, 2, 16, 10),
    }
    for name, (tn, n, steps, seed, ml, pe) in cfgs.items():
        r = rollout(tn, n, steps, seed, ml, True, pe)
        np.savez_compressed(os.path.join(OUT, f"rollout_{name}.npz"), tier=tn, n=n, steps=steps,
                            seed=seed, max_len=ml or 0, pix_every=pe, **r)

    # ---- engine-level fuzz: scrambled states exercise rare branches
    for tn, n, steps, seed in (("extended", 48, 60, 11), ("classic", 48, 60, 12)):
        t = tiers[tn]
        rng = np.random.default_rng(seed)
        bs = batch_reset(BatchConfig(n_envs=n, tier=t), seed)
        sim = bs.sim
        scramble(sim, rng, tn)
        start = {f: getattr(sim, f).copy() for f in FIELD_NAMES}
        ws = Workspace(n, t.n_achievements)
        actions = rng.integers(0, t.n_actions, (steps, n)).astype(np.int64)
        rec = {k: [] for k in ("state", "reward", "done", "newly", "obs", "pix")}
        px = 7 if tn == "classic" else 10
        for k in range(steps):
            rw, dn, nw, _ = step_batch(sim, actions[k], ws)
            rec["state"].append(state_digest({f: getattr(sim, f) for f in FIELD_NAMES}, FIELD_NAMES))
            rec["reward"].append(digest(rw))
            rec["done"].append(digest(dn))
            rec["newly"].append(digest(nw))
            rec["obs"].append(digest(encode_symbolic_batch(sim)))
            frames = np.stack([render_tiles(GameState(sim.view(slice(i, i + 1))), px) for i in range(n)])
            rec["pix"].append(digest(frames))
            if dn.any():  # revive finished envs (engine-level fuzz, no pool)
                sim.health[dn] = 5.0
                sim.time[dn] = 0
                sim.done[dn] = False
        np.savez_compressed(os.path.join(OUT, f"fuzz_{tn}.npz"), tier=tn, n=n, actions=actions,
                            **{f"start_{f}": v for f, v in start.items()},
                            **{k: np.array(v, np.uint64) for k, v in rec.items()})

    # ---- the recorded 500-action session (frontend fixture), engine-direct
    fx = json.load(open("/root/reference/pkg/frontend/test/fixtures/session_500.json"))
    steps_out = []
    state = None

    def episode(seed):
        world = generate_world(make_level_params(seed), EXTENDED)
        return reset(world, EXTENDED, R.make_stream(seed))

    state = episode(fx["seed"])
    for entry in fx["steps"]:
        if entry["action"] is None:
            state = episode(entry["reset_seed"])
            steps_out.append({"reset_seed": entry["reset_seed"]})
            continue
        out = step(state, entry["action"])
        state = out.state
        steps_out.append({"action": entry["action"], "reward": out.reward, "done": out.done,
                          "state": state_digest({f: getattr(state.sim, f) for f in FIELD_NAMES},
                                                FIELD_NAMES)})
    json.dump({"seed": fx["seed"], "steps": steps_out}, open(os.path.join(OUT, "session.json"), "w"))

    meta = {"numpy": np.__version__, "python": sys.version.split()[0],
            "simd": __import__("numpy._core._multiarray_umath", fromlist=["x"]).__cpu_features__,
            "generator": "tests/golden/make_golden.py", "reference": REF}
    meta["simd"] = sorted(k for k, v in meta["simd"].items() if v)
    json.dump(meta, open(os.path.join(OUT, "meta.json"), "w"), indent=1)
    print("goldens written to", OUT)


if __name__ == "__main__":
    main()
