"""Mint game_state blobs with the reference's serializer (run HERE, where /root/reference exists).

    python tests/golden/make_serialize_golden.py

For each tier, a reference GameState (engine.reset on a generated world,
then random-policy engine.step until step 60 or the episode ends) is written
with the unmodified ``gridrogue.serialize.state_to_bytes``
(serialize.py:155-159) to ``game_state_<tier>.bin``, and a 4-env SimState
after 40 batch steps to ``game_state_<tier>_batch.bin``.  tests/test_gpu.py
loads them into device batches with paper_2402_16801_b200.serialize.
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


if __name__ == "__main__":
    main()
