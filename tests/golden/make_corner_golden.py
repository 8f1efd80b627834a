"""Mint goldens for the numpy corners of worldgen (run HERE, with the reference).

    python tests/golden/make_corner_golden.py

Writes tests/golden/numpy_corners.npz:

* ``argsort6_digest`` -- ``np.argsort`` (the reference's call,
  worldgen.py:647-649: default kind, float32, 6 elements) over all 6^6 value
  patterns in {0..5}: every tie configuration of six keys.  numpy >= 2 runs it
  through x86-simd-sort's AVX-512 bitonic network, which is not stable.
* ``tie_seeds`` / ``tie_potion`` / ``tie_world`` -- LevelParams seeds whose six
  potion draws ``vuniform32(u32(hash2(seed, 42)), 0..5)`` contain equal values
  and whose numpy order differs from a stable sort, with the reference's
  ``generate_world(make_level_params(seed), EXTENDED)`` potion permutation and
  a digest of the whole world (maps, ladders, chests), as worlds.npz does.
* ``trig_x`` / ``trig_digest`` -- float32 angles in [0, 2*pi]
  (the cave gradients, perlin.py:71-72 with worldgen.py:424's float64 dtype)
  where numpy's float64 sin or cos (glibc) is NOT the correctly rounded value
  (a long-double evaluation rounded to double disagrees), every 4th one, with
  digests of numpy's results.

Writes tests/golden/template_worlds.npz: ``generate_world`` with the
reference's ``worldgen.MAX_GEN_RETRIES`` set to 0 at run time (the module is
not edited), so every floor is ``_template_floor`` (worldgen.py:549-595) and
the chests / potions are assigned over the templates; arrays in
``LevelBuffer.world`` layout.
"""

from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
from tests._digest import digest  # noqa: E402


def world_digest(w) -> int:
    parts = []
    for fm in w.floors:
        parts += [fm.blocks, fm.items, np.array(fm.spawn, np.int64),
                  np.array(fm.ladder_down or (-1, -1), np.int64),
                  np.array(fm.ladder_up or (-1, -1), np.int64)]
    ch = np.array([c for lanes in w.chests for c in lanes] or np.zeros((0, 4)), np.int64)
    return digest(digest(*parts), digest(ch.reshape(-1, 4)))


def main() -> None:
    sys.path.insert(0, REF)
    from gridrogue import EXTENDED, make_level_params, generate_world
    from gridrogue import rng as R

    pats = np.array(list(itertools.product(range(6), repeat=6)), np.float32)
    order = np.stack([np.argsort(p) for p in pats]).astype(np.int64)

    seeds, potions, worlds = [], [], []
    base, chunk = 0, 1 << 22
    while len(seeds) < 24:     # vectorised search over seeds, then per-seed checks
        cand = np.arange(base, base + chunk, dtype=np.uint64)
        keys = (R.vhash2(cand, np.uint64(42)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        v = np.stack([R.vuniform32(keys, np.uint32(i)) for i in range(6)], 1)
        vs = np.sort(v, 1)
        for s in cand[(vs[:, 1:] == vs[:, :-1]).any(1)].tolist():
            v6 = R.vuniform32(np.uint32(R.hash2(s, 42) & 0xFFFFFFFF), np.arange(6, dtype=np.uint32))
            if np.array_equal(np.argsort(v6), np.argsort(v6, kind="stable")) or len(seeds) >= 24:
                continue
            w = generate_world(make_level_params(s), EXTENDED)
            seeds.append(s)
            potions.append(w.potion_permutation.astype(np.uint8))
            worlds.append(world_digest(w))
        base += chunk
    print("tie seeds", seeds)

    # glibc float64 sin / cos: the hard cases
    lo, hi = np.float32(0).view(np.uint32), np.float32(2 * np.pi).view(np.uint32)
    hard = []
    for a in range(int(lo), int(hi) + 1, 1 << 25):
        x = np.arange(a, min(a + (1 << 25), int(hi) + 1), dtype=np.uint32).view(np.float32)
        xd, xl = x.astype(np.float64), x.astype(np.longdouble)
        bad = (np.sin(xd) != np.sin(xl).astype(np.float64)) | (np.cos(xd) != np.cos(xl).astype(np.float64))
        hard.append(x[bad])
    hx = np.concatenate(hard)[::4]
    print("hard trig inputs kept", len(hx))
    np.savez_compressed(os.path.join(OUT, "numpy_corners.npz"),
                        argsort6_digest=np.uint64(digest(order)), argsort6_sample=order[::97],
                        tie_seeds=np.array(seeds, np.uint64), tie_potion=np.stack(potions),
                        tie_world=np.array(worlds, np.uint64),
                        trig_x=hx, trig_digest=np.array([digest(np.sin(hx.astype(np.float64))),
                                                         digest(np.cos(hx.astype(np.float64)))], np.uint64),
                        meta=json.dumps({"numpy": np.__version__}))
    template_worlds()


TEMPLATE_SEEDS = {"classic": [0, 7], "extended": [0, 7, 123]}


def template_worlds() -> None:
    from gridrogue import CLASSIC, EXTENDED, make_level_params, generate_world
    from gridrogue import worldgen
    out = {}
    saved = worldgen.MAX_GEN_RETRIES
    worldgen.MAX_GEN_RETRIES = 0
    try:
        for tname, tier in (("classic", CLASSIC), ("extended", EXTENDED)):
            for seed in TEMPLATE_SEEDS[tname]:
                w = generate_world(make_level_params(seed), tier)
                tag = f"{tname}_{seed}"
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
                out[f"{tag}_digest"] = np.uint64(world_digest(w))
    finally:
        worldgen.MAX_GEN_RETRIES = saved
    np.savez_compressed(os.path.join(OUT, "template_worlds.npz"), **out)


if __name__ == "__main__":
    main()
