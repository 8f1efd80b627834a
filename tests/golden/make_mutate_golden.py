"""Mint UED level goldens from the reference (run HERE, where /root/reference exists).

    python tests/golden/make_mutate_golden.py

For a few seeds per tier, with the unmodified reference:
  params  = worldgen.make_level_params(seed)                    (worldgen.py:75-87)
  noisy   = mutate.mutate_noise(params, make_stream(seed + 1))  (mutate.py:36-44)
  world   = worldgen.generate_world(noisy, tier)                (worldgen.py:636-651)
  swapped = mutate.mutate_swap(world, make_stream(seed + 2))    (mutate.py:58-72)
  rswap   = mutate.mutate_rswap(world, make_stream(seed + 3))   (mutate.py:75-103)
  state   = engine.reset(rswap, tier, make_stream(seed + 4))    (engine.py:749-758)
and writes every array to ``ued_levels.npz`` next to this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
SEEDS = {"classic": [3, 1001], "extended": [5, 77, 2024]}


def main() -> None:
    sys.path.insert(0, REF)
    from gridrogue import CLASSIC, EXTENDED, make_level_params, generate_world
    from gridrogue import rng as R
    from gridrogue import engine
    from gridrogue.mutate import mutate_noise, mutate_swap, mutate_rswap
    from gridrogue.state import FIELD_NAMES
    tiers = {"classic": CLASSIC, "extended": EXTENDED}
    out = {}

    def put_params(tag, p):
        out[f"{tag}_seed"] = np.uint64(p.seed)
        out[f"{tag}_angles"] = np.concatenate([a.reshape(-1) for a in p.overworld_angles]).astype(np.float32)
        out[f"{tag}_floor_seeds"] = np.array(p.per_floor_seeds, np.uint64)

    def put_world(tag, w):
        out[f"{tag}_blocks"] = np.stack([f.blocks for f in w.floors])
        out[f"{tag}_items"] = np.stack([f.items for f in w.floors])
        out[f"{tag}_spawn"] = np.array(w.floors[0].spawn, np.int16)
        out[f"{tag}_ladders"] = np.array([[*(f.ladder_down or (-1, -1)), *(f.ladder_up or (-1, -1))]
                                          for f in w.floors], np.int16)
        out[f"{tag}_potion"] = w.potion_permutation.astype(np.uint8)
        ch = np.full((len(w.floors), 6, 4), -1, np.int64)
        for f, lanes in enumerate(w.chests):
            for j, c in enumerate(lanes):
                ch[f, j] = c
        out[f"{tag}_chests"] = ch

    for tname, seeds in SEEDS.items():
        tier = tiers[tname]
        for seed in seeds:
            tag = f"{tname}_{seed}"
            p = make_level_params(seed)
            put_params(f"{tag}_params", p)
            noisy = mutate_noise(p, R.make_stream(seed + 1))
            put_params(f"{tag}_noisy", noisy)
            world = generate_world(noisy, tier)
            put_world(f"{tag}_world", world)
            put_world(f"{tag}_swap", mutate_swap(world, R.make_stream(seed + 2)))
            rs = mutate_rswap(world, R.make_stream(seed + 3))
            put_world(f"{tag}_rswap", rs)
            st = engine.reset(rs, tier, R.make_stream(seed + 4))
            out[f"{tag}_install_key"] = np.uint64(R.split(R.make_stream(seed + 4), 0).key)
            for f in FIELD_NAMES:
                out[f"{tag}_state_{f}"] = getattr(st.sim, f)
            print(tag, "ok", flush=True)
    np.savez_compressed(os.path.join(OUT, "ued_levels.npz"), **out)


if __name__ == "__main__":
    main()
