"""Mint game_state blobs with the reference's serializer (run HERE, where /root/reference exists).

    python tests/golden/make_serialize_golden.py

For each tier, a reference GameState (engine.reset on a generated world,
then random-policy engine.step until step 60 or the episode ends) is written
with the unmodified ``gridrogue.serialize.state_to_bytes``
(serialize.py:155-159) to ``game_state_<tier>.bin``, and a 4-env SimState
after 40 batch steps to ``game_state_<tier>_batch.bin``.  tests/test_gpu.py
loads them into device batches with paper_2402_16801_b200.serialize.

The level formats (serialize.py:43-151), written by the reference's own
``params_to_bytes`` / ``params_to_json`` / ``world_to_bytes`` /
``world_to_json``:
  level_params_77.bin / .json       make_level_params(77)
  level_params_noisy_77.bin         mutate_noise(make_level_params(77), make_stream(78))
  world_<tag>.bin (+ .json for classic_3): generate_world for classic_3 and
  extended_77, the extended_5 world after mutate_rswap, and extended_7 with
  MAX_GEN_RETRIES patched to 0 at run time (every floor a template); and
  world_<tag>_installed.npz: engine.reset(world, tier, make_stream(seed + 4))
  -- the SimState an env holds after install_world with that key.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from gridrogue import CLASSIC, EXTENDED, make_level_params, generate_world
    from gridrogue import rng as R
    from gridrogue import engine
    from gridrogue.batch import BatchConfig, batch_reset, batch_step
    from gridrogue.policies import RandomPolicy
    from gridrogue.serialize import state_to_bytes
    from gridrogue.state import GameState
    for tier in (CLASSIC, EXTENDED):
        world = generate_world(make_level_params(1234), tier)
        st = engine.reset(world, tier, R.make_stream(99))
        pol = RandomPolicy(7, tier.n_actions)
        for t in range(60):
            a = int(pol.actions_at(t, 1)[0]) if hasattr(pol, "actions_at") else int(pol.actions(st.sim)[0])
            out = engine.step(st, a)
            st = out.state
            if out.done:
                break
        with open(os.path.join(OUT, f"game_state_{tier.name}.bin"), "wb") as fh:
            fh.write(state_to_bytes(st))
        bs = batch_reset(BatchConfig(n_envs=4, tier=tier), 5)
        pol = RandomPolicy(5, tier.n_actions)
        for _ in range(40):
            bs, _ = batch_step(bs, pol.actions(bs.sim))
        with open(os.path.join(OUT, f"game_state_{tier.name}_batch.bin"), "wb") as fh:
            fh.write(state_to_bytes(GameState(bs.sim)))
        print(tier.name, "ok")
    levels()


def levels() -> None:
    import json
    from gridrogue import CLASSIC, EXTENDED, make_level_params, generate_world
    from gridrogue import rng as R
    from gridrogue import engine, worldgen
    from gridrogue.mutate import mutate_noise, mutate_rswap
    from gridrogue.serialize import params_to_bytes, params_to_json, world_to_bytes, world_to_json
    from gridrogue.state import FIELD_NAMES

    def put(name, blob):
        with open(os.path.join(OUT, name), "wb") as fh:
            fh.write(blob)

    p = make_level_params(77)
    put("level_params_77.bin", params_to_bytes(p))
    json.dump(params_to_json(p), open(os.path.join(OUT, "level_params_77.json"), "w"))
    put("level_params_noisy_77.bin", params_to_bytes(mutate_noise(p, R.make_stream(78))))

    def world(tag, w, tier, seed, with_json=False):
        put(f"world_{tag}.bin", world_to_bytes(w))
        if with_json:
            json.dump(world_to_json(w), open(os.path.join(OUT, f"world_{tag}.json"), "w"))
        st = engine.reset(w, tier, R.make_stream(seed + 4))
        np.savez_compressed(os.path.join(OUT, f"world_{tag}_installed.npz"),
                            key=np.uint64(R.split(R.make_stream(seed + 4), 0).key),
                            **{f: getattr(st.sim, f) for f in FIELD_NAMES})

    world("classic_3", generate_world(make_level_params(3), CLASSIC), CLASSIC, 3, with_json=True)
    world("extended_77", generate_world(p, EXTENDED), EXTENDED, 77)
    w5 = generate_world(make_level_params(5), EXTENDED)
    world("extended_rswap_5", mutate_rswap(w5, R.make_stream(8)), EXTENDED, 5)
    saved = worldgen.MAX_GEN_RETRIES
    worldgen.MAX_GEN_RETRIES = 0
    try:
        world("extended_template_7", generate_world(make_level_params(7), EXTENDED), EXTENDED, 7)
    finally:
        worldgen.MAX_GEN_RETRIES = saved
    print("levels ok")


if __name__ == "__main__":
    main()
