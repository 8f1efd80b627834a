"""State scrambler for the engine-level fuzz goldens (used by make_golden.py).

Randomises inventories, attributes, floors, boss phases, nearby stations,
creatures, projectiles and plants of a reference SimState in place so that a
short rollout exercises the rare branches of engine.py / creatures.py
(enchanting, potions, ladders, boss waves, projectile hits) that a uniform
random policy from a fresh world almost never reaches.
"""

import numpy as np


def scramble(sim, rng, tier):
    n = sim.n
    ext = tier == "extended"
    for name in ("inv_wood","inv_stone","inv_coal","inv_iron","inv_diamond","inv_sapphire","inv_ruby","inv_sapling","inv_torch","inv_arrow","inv_book"):
        getattr(sim, name)[:] = rng.integers(0, 12, n) * (rng.random(n) < 0.7)
    sim.inv_potion[:] = rng.integers(0, 3, (n, 6))
    sim.pick_tier[:] = rng.integers(0, 5, n); sim.sword_tier[:] = rng.integers(0, 5, n)
    if ext:
        sim.has_bow[:] = rng.random(n) < 0.6
        sim.learned_fire[:] = rng.random(n) < 0.5; sim.learned_ice[:] = rng.random(n) < 0.4
        sim.mana[:] = rng.integers(0, 18, n).astype(np.float32)
        sim.xp[:] = rng.integers(0, 4, n); sim.dex[:] = rng.integers(1, 6, n); sim.str_[:] = rng.integers(1, 6, n); sim.intel[:] = rng.integers(1, 6, n)
        sim.armour[:] = rng.integers(0, 3, (n, 4)); sim.armour_ench[:] = rng.integers(0, 3, (n, 4)) * (rng.random((n,4)) < 0.3)
        sim.sword_ench[:] = rng.integers(0, 3, n); sim.bow_ench[:] = rng.integers(0, 3, n)
        # teleport to a random floor at its up ladder
        fl = rng.integers(0, 9, n)
        for i in range(n):
            f = int(fl[i])
            if f == 0: continue
            sim.pfloor[i] = f; sim.prow[i], sim.pcol[i] = sim.ladder_up[i, f]
            sim.floors_visited[i, :f+1] = rng.random(f+1) < 0.7; sim.floors_visited[i, 0] = True
            if f == 8:
                sim.boss_wave[i] = rng.integers(0, 9); sim.boss_vuln[i] = rng.random() < 0.4
                sim.boss_timer[i] = rng.integers(1, 21); sim.boss_hp[i] = np.float32(rng.integers(1, 61))
                if sim.boss_vuln[i]:
                    sim.blocks[i, 8, sim.necro_pos[i,0], sim.necro_pos[i,1]] = 36
                    # put the player in front of the necromancer sometimes
                    if rng.random() < 0.5:
                        sim.prow[i] = sim.necro_pos[i,0] + 1; sim.pcol[i] = sim.necro_pos[i,1]; sim.facing[i] = 2
    sim.health[:] = rng.integers(1, 10, n).astype(np.float32)
    sim.food[:] = rng.integers(0, 14, n).astype(np.float32); sim.drink[:] = rng.integers(0, 14, n).astype(np.float32)
    sim.energy[:] = rng.integers(0, 14, n).astype(np.float32)
    sim.sleeping[:] = rng.random(n) < 0.1
    if ext: sim.resting[:] = rng.random(n) < 0.05
    sim.time[:] = rng.integers(0, 2000, n)
    sim.clocks[:] = rng.integers(0, 40, (n, 6))
    sim.facing[:] = rng.integers(0, 4, n)
    # sprinkle stations / torches / creatures near the player
    F = sim.blocks.shape[1]; H = sim.blocks.shape[2]
    for i in range(n):
        f = int(sim.pfloor[i]); r, c = int(sim.prow[i]), int(sim.pcol[i])
        for _ in range(6):
            dr, dc = rng.integers(-2, 3, 2)
            rr, cc = r + dr, c + dc
            if 0 <= rr < H and 0 <= cc < H and (dr or dc):
                choices = [11, 12, 5, 4, 8, 9, 10, 3, 16, 15, 2, 7] + ([30, 31, 23, 21, 22, 24, 20] if ext else [])
                sim.blocks[i, f, rr, cc] = rng.choice(choices)
                if ext and rng.random() < 0.2: sim.items[i, f, rr, cc] = 1
        for cls, cap in (("mel", 3), ("ran", 2), ("pas", 3)):
            for l in range(cap):
                if rng.random() < 0.5:
                    pos = getattr(sim, cls + "_pos"); pos[i, f, l] = (r + rng.integers(-7, 8), c + rng.integers(-7, 8))
                    kinds = {"mel": [0,3,6,9,11,13,15,17], "ran": [1,4,7,10,12,14,16,18], "pas": [2,5,8]}[cls]
                    k = kinds[f] if (f < 8 and cls != "pas") else rng.choice(kinds)
                    if tier == "classic": k = {"mel": 0, "ran": 1, "pas": 2}[cls]
                    getattr(sim, cls + "_type")[i, f, l] = k
                    getattr(sim, cls + "_alive")[i, f, l] = True
                    getattr(sim, cls + "_hp")[i, f, l] = np.float32(rng.integers(1, 8))
                    if cls != "pas": getattr(sim, cls + "_cd")[i, f, l] = rng.integers(0, 4)
        if ext:
            for l in range(3):
                if rng.random() < 0.3:
                    sim.pproj_alive[i, l] = True; sim.pproj_pos[i, l] = (r + rng.integers(-3, 4), c + rng.integers(-3, 4))
                    sim.pproj_dir[i, l] = rng.integers(0, 4); sim.pproj_type[i, l] = rng.integers(0, 3); sim.pproj_ttl[i, l] = rng.integers(1, 7)
                    sim.pproj_dmg[i, l] = rng.integers(0, 8, 3).astype(np.float32)
        for l in range(3):
            if rng.random() < 0.3:
                sim.eproj_alive[i, l] = True; sim.eproj_pos[i, l] = (r + rng.integers(-3, 4), c + rng.integers(-3, 4))
                sim.eproj_dir[i, l] = rng.integers(0, 4); sim.eproj_type[i, l] = rng.integers(3, 9); sim.eproj_ttl[i, l] = rng.integers(1, 7)
                sim.eproj_dmg[i, l] = rng.integers(0, 6, 3).astype(np.float32)
        if f == 0:
            for l in range(10):
                if rng.random() < 0.3:
                    pr, pc = r + rng.integers(-3, 4), c + rng.integers(-3, 4)
                    if 0 <= pr < H and 0 <= pc < H:
                        sim.plant_alive[i, l] = True; sim.plant_pos[i, l] = (pr, pc); sim.plant_age[i, l] = rng.integers(0, 70)
                        sim.blocks[i, 0, pr, pc] = rng.choice([15, 16])
