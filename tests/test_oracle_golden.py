"""Pin the C oracle to golden vectors minted from the numpy reference.

The goldens (tests/golden/*.npz, made by tests/golden/make_golden.py from the
unmodified reference) cover rng.py, numpy's float32 sin/cos, worldgen for 520
seeds, BatchEnv-semantics rollouts (state, reward, done, newly, info, symbolic
obs, pixel frames) for both tiers including reset-stress runs, engine-level
fuzz from scrambled states, and the reference's recorded 500-action session.
"""

import json
import os

import numpy as np
import pytest

from tests._digest import digest, state_digest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_rng_known_answers(oracle_lib):
    O = oracle_lib
    g = np.load(os.path.join(GOLD, "rng.npz"))
    L = O.lib()
    for i, k in enumerate(g["keys"]):
        for j, c in enumerate(g["ctrs"]):
            assert L.go_hash2(int(k), int(c)) == int(g["hash2"][i, j])
    v = np.array([L.go_vuniform32(0x1234567, i) for i in range(4096)], np.float32)
    assert np.array_equal(v, g["vuniform32"])


def test_numpy_f32_sincos_restatement(oracle_lib):
    """Hazard H1: numpy's SIMD float32 sin/cos, restated, bit-exact."""
    L = oracle_lib.lib()
    g = np.load(os.path.join(GOLD, "rng.npz"))
    xs = (np.arange(200_000, dtype=np.float64) * (2 * np.pi / 200_000)).astype(np.float32)
    s = np.array([L.go_np_sinf(float(x)) for x in xs], np.float32)
    c = np.array([L.go_np_cosf(float(x)) for x in xs], np.float32)
    assert digest(s) == int(g["trig_digest"][0])
    assert digest(c) == int(g["trig_digest"][1])


@pytest.mark.parametrize("tier,count", [("classic", 400), ("extended", 120)])
def test_worldgen_matches_reference(oracle_lib, tier, count):
    O = oracle_lib
    g = np.load(os.path.join(GOLD, "worlds.npz"))[tier]
    assert len(g) == count
    for seed in range(count):
        w = O.generate_world(seed, tier)
        parts = []
        for f in range(len(w["blocks"])):
            ld = w["ladder_down"][f].astype(np.int64)
            lu = w["ladder_up"][f].astype(np.int64)
            parts += [w["blocks"][f], w["items"][f],
                      np.array(w["spawn"] if f == 0 else _floor_spawn(w, f), np.int64), ld, lu]
        ch = np.array([c for lanes in w["chests"] for c in lanes] or np.zeros((0, 4)), np.int64)
        assert digest(*parts) == int(g[seed, 0]), f"{tier} seed {seed} maps"
        assert digest(ch.reshape(-1, 4)) == int(g[seed, 1]), f"{tier} seed {seed} chests"
        assert digest(w["potion"].astype(np.int64)) == int(g[seed, 2]), f"{tier} seed {seed} potion"


def _floor_spawn(w, f):
    # FloorMap.spawn of lower floors is their up ladder (worldgen.py:406,468,520,546)
    lu = w["ladder_up"][f]
    return (int(lu[0]), int(lu[1]))


ROLLOUTS = sorted(f[len("rollout_"):-4] for f in os.listdir(GOLD) if f.startswith("rollout_"))


@pytest.mark.parametrize("name", ROLLOUTS)
def test_batch_rollout_matches_reference(oracle_lib, name):
    """BatchEnv semantics: batch_step + post-reset obs, random policy."""
    O = oracle_lib
    g = np.load(os.path.join(GOLD, f"rollout_{name}.npz"))
    tier, n, steps, seed = str(g["tier"]), int(g["n"]), int(g["steps"]), int(g["seed"])
    ml = int(g["max_len"]) or None
    pe = int(g["pix_every"])
    b = O.OracleBatch(tier, n, seed, max_episode_length=ml)
    st = b.state
    assert state_digest(st.export_fields(), O.FIELD_NAMES) == int(g["reset"][0])
    assert digest(st.encode_symbolic()) == int(g["reset"][1])
    na = O.TIERS[tier]["NA"]
    px = 7 if tier == "classic" else 10
    for k in range(steps):
        a = O.random_actions(seed, k, n, na)
        r, d, nw, info = b.step(a)
        assert digest(r) == int(g["reward"][k]), f"reward step {k}"
        assert digest(d) == int(g["done"][k]), f"done step {k}"
        assert digest(nw) == int(g["newly"][k]), f"newly step {k}"
        assert digest(info["time"], info["floor"]) == int(g["info"][k]), f"info step {k}"
        assert state_digest(st.export_fields(), O.FIELD_NAMES) == int(g["state"][k]), f"state step {k}"
        assert digest(st.encode_symbolic()) == int(g["obs"][k]), f"obs step {k}"
        if pe and k % pe == 0:
            assert digest(st.render_pixels(px)) == int(g["pix"][k]), f"pixels step {k}"
    ex = st.export_fields()
    for f, dg in zip(O.FIELD_NAMES, g["final_fields"]):
        assert digest(ex[f]) == int(dg), f
    s = b.stats()
    assert s["episodes"] == int(g["episodes"]) and s["total_steps"] == int(g["total_steps"])
    assert np.array_equal(s["ach_episodes"], g["ach_episodes"])
    assert np.array_equal(ex["params_seed"], g["level_seeds"])


@pytest.mark.parametrize("tier", ["classic", "extended"])
def test_engine_fuzz_matches_reference(oracle_lib, tier):
    """Scrambled start states: enchanting, potions, ladders, boss, projectiles."""
    O = oracle_lib
    g = np.load(os.path.join(GOLD, f"fuzz_{tier}.npz"))
    n = int(g["n"])
    st = O.OracleState(tier, n)
    st.import_fields({f: g[f"start_{f}"] for f in O.FIELD_NAMES})
    px = 7 if tier == "classic" else 10
    for k, a in enumerate(g["actions"]):
        r, d, nw, _ = st.step(a)
        ex = st.export_fields()
        assert digest(r) == int(g["reward"][k]), f"reward step {k}"
        assert digest(d) == int(g["done"][k]), f"done step {k}"
        assert digest(nw) == int(g["newly"][k]), f"newly step {k}"
        assert state_digest(ex, O.FIELD_NAMES) == int(g["state"][k]), f"state step {k}"
        assert digest(st.encode_symbolic()) == int(g["obs"][k]), f"obs step {k}"
        assert digest(st.render_pixels(px)) == int(g["pix"][k]), f"pixels step {k}"
        if d.any():
            ex["health"][d] = 5.0
            ex["time"][d] = 0
            ex["done"][d] = False
            st.import_fields(ex)


def test_recorded_session_replay(oracle_lib):
    """The reference's 500-action session (all 43 actions, 3 resets)."""
    O = oracle_lib
    g = json.load(open(os.path.join(GOLD, "session.json")))

    def episode(seed):
        st = O.OracleState("extended", 1)
        key = O.lib().go_hash2(O.lib().go_mix(seed), O.lib().go_hash2(0, 0))
        st.install_seed(0, seed, key)
        return st

    st = episode(g["seed"])
    used = set()
    for e in g["steps"]:
        if "reset_seed" in e:
            st = episode(e["reset_seed"])
            continue
        used.add(e["action"])
        r, d, _, _ = st.step(np.array([e["action"]]))
        assert float(r[0]) == e["reward"]
        assert bool(d[0]) == e["done"]
        assert state_digest(st.export_fields(), O.FIELD_NAMES) == e["state"]
    assert used == set(range(43))


LONG = sorted(f[len("long_"):-4] for f in os.listdir(GOLD) if f.startswith("long_"))


@pytest.mark.parametrize("name", LONG)
def test_long_rollout_matches_reference(oracle_lib, name):
    if name.endswith("_n1024") and not os.environ.get("GR_SLOW"):
        pytest.skip("10^7 env-steps on the oracle: set GR_SLOW=1 (~1 min, 8 cores)")
    """BASELINE.json north star: 10^4-step random rollouts of all four variants
    (tests/golden/make_long_golden.py, minted from the unmodified reference):
    every step's reward / done / observation, the full SimState + f64 episode
    accumulators every 2,500 steps, the final fields and EpisodeStats."""
    O = oracle_lib
    g = np.load(os.path.join(GOLD, f"long_{name}.npz"))
    tier, obs_mode, n = str(g["tier"]), str(g["obs_mode"]), int(g["n"])
    steps, seed, ml, every, px = (int(g[k]) for k in ("steps", "seed", "max_len", "every", "tile_px"))
    obs_every = int(g["obs_every"]) if "obs_every" in g.files else 1
    b = O.OracleBatch(tier, n, seed, max_episode_length=ml or None, threads=8 if n > 256 else 1)
    st = b.state

    def observe():
        return st.encode_symbolic() if obs_mode == "symbolic" else st.render_pixels(px)

    assert state_digest(st.export_fields(), O.FIELD_NAMES) == int(g["reset"][0])
    assert digest(observe()) == int(g["reset"][1])
    na = O.TIERS[tier]["NA"]
    c = 0
    for k in range(steps):
        r, d, _, _ = b.step(O.random_actions(seed, k, n, na))
        assert digest(r.astype(np.float32)) == int(g["reward"][k]), f"reward step {k}"
        assert digest(d) == int(g["done"][k]), f"done step {k}"
        if k % obs_every == 0:
            assert digest(observe()) == int(g["obs"][k]), f"obs step {k}"
        if (k + 1) % every == 0:
            assert state_digest(st.export_fields(), O.FIELD_NAMES) == int(g["ckpt"][c][0]), f"state step {k}"
            assert digest(*b.episode_progress()) == int(g["ckpt"][c][1]), f"episode acc step {k}"
            c += 1
    ex = st.export_fields()
    for f, dg in zip(O.FIELD_NAMES, g["final_fields"]):
        assert digest(ex[f]) == int(dg), f
    s = b.stats()
    assert s["episodes"] == int(g["episodes"]) and s["total_steps"] == int(g["total_steps"])
    assert np.array_equal(s["ach_episodes"], g["ach_episodes"])
    assert np.array_equal(ex["params_seed"], g["level_seeds"])


@pytest.mark.skipif(not os.environ.get("GR_SLOW"), reason="65,536-env oracle run: set GR_SLOW=1 (~2 min, 8 cores)")
def test_north_star_size_matches_reference(oracle_lib):
    """The bench workload (65,536 extended envs) on the oracle against the
    reference's digests -- the same fixture tests/test_gpu.py checks the CUDA
    path against."""
    O = oracle_lib
    g = np.load(os.path.join(GOLD, "north_star_ext_n65536.npz"))
    n, seed, steps = int(g["n"]), int(g["seed"]), int(g["steps"])
    b = O.OracleBatch("extended", n, seed, threads=os.cpu_count() or 8)
    st = b.state
    assert state_digest(st.export_fields(), O.FIELD_NAMES) == int(g["reset"][0])
    assert digest(st.encode_symbolic()) == int(g["reset"][1])
    for k in range(steps):
        r, d, nw, info = b.step(O.random_actions(seed, k, n, 43))
        assert digest(r.astype(np.float32)) == int(g["reward"][k]), f"reward step {k}"
        assert digest(d) == int(g["done"][k]), f"done step {k}"
        assert digest(nw) == int(g["newly"][k]), f"newly step {k}"
        assert digest(info["time"], info["floor"]) == int(g["info"][k]), f"info step {k}"
        assert digest(st.encode_symbolic()) == int(g["obs"][k]), f"obs step {k}"
        assert state_digest(st.export_fields(), O.FIELD_NAMES) == int(g["state"][k]), f"state step {k}"
    assert digest(*b.episode_progress()) == int(g["episode_acc"])
    assert digest(st.export_fields()["params_seed"]) == int(g["level_seeds_digest"])


def _corners():
    return np.load(os.path.join(GOLD, "numpy_corners.npz"))


def test_numpy_argsort6_tie_order(oracle_lib):
    """worldgen.py:647-649: np.argsort's (unstable, AVX-512 network) order on
    every tie pattern of six float32 keys (tests/golden/make_corner_golden.py)."""
    import itertools
    L = oracle_lib.lib()
    pats = np.array(list(itertools.product(range(6), repeat=6)), np.float32)
    out = np.zeros(pats.shape, np.uint8)
    for i in range(len(pats)):
        L.go_np_argsort6(pats[i].ctypes.data, out[i].ctypes.data)
    g = _corners()
    assert np.array_equal(out[::97].astype(np.int64), g["argsort6_sample"])
    assert digest(out.astype(np.int64)) == int(g["argsort6_digest"])
    stable = np.argsort(pats, axis=1, kind="stable")
    assert (out != stable).any(axis=1).sum() > 1000     # really not a stable sort


def test_potion_ties_match_reference(oracle_lib):
    """Worlds whose potion draws tie: the reference's permutation and world."""
    O = oracle_lib
    g = _corners()
    for s, pot, wd in zip(g["tie_seeds"], g["tie_potion"], g["tie_world"]):
        w = O.generate_world(int(s), "extended")
        assert np.array_equal(w["potion"], pot), f"seed {s}"
        parts = []
        for f in range(len(w["blocks"])):
            parts += [w["blocks"][f], w["items"][f],
                      np.array(w["spawn"] if f == 0 else _floor_spawn(w, f), np.int64),
                      w["ladder_down"][f].astype(np.int64), w["ladder_up"][f].astype(np.int64)]
        ch = np.array([c for lanes in w["chests"] for c in lanes] or np.zeros((0, 4)), np.int64)
        assert digest(digest(*parts), digest(ch.reshape(-1, 4))) == int(wd), f"seed {s} world"


def test_template_floors_match_reference(oracle_lib):
    """worldgen.py:549-595: with MAX_GEN_RETRIES = 0 every floor is the
    _template_floor fallback; chests and potions are assigned over them
    (tests/golden/template_worlds.npz, minted with the reference's constant
    patched at run time)."""
    O = oracle_lib
    L = O.lib()
    g = np.load(os.path.join(GOLD, "template_worlds.npz"))
    tags = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_digest")})
    assert len(tags) == 5
    L.go_set_max_gen_retries(0)
    try:
        for tag in tags:
            tier, seed = tag.split("_")
            w = O.generate_world(int(seed), tier)
            assert np.array_equal(np.stack(w["blocks"]), g[f"{tag}_blocks"]), tag
            assert np.array_equal(np.stack(w["items"]), g[f"{tag}_items"]), tag
            assert np.array_equal(w["potion"], g[f"{tag}_potion"]), tag
            lad = np.concatenate([np.asarray(w["ladder_down"]), np.asarray(w["ladder_up"])], axis=1)
            assert np.array_equal(lad.astype(np.int16), g[f"{tag}_ladders"]), tag
            ch = np.full(g[f"{tag}_chests"].shape, -1, np.int64)
            for f, lanes in enumerate(w["chests"]):
                for j, c in enumerate(lanes):
                    ch[f, j] = c
            assert np.array_equal(ch, g[f"{tag}_chests"]), tag
    finally:
        L.go_set_max_gen_retries(16)


@pytest.mark.parametrize("tier", ["classic", "extended"])
def test_pixels_every_tile_size_match_reference(oracle_lib, tier):
    """tiles.render_tiles at every supported tile size (7, 10, 16 px), both
    tiers, 120 auto-resetting steps (tests/golden/pixels_px.npz)."""
    O = oracle_lib
    g = np.load(os.path.join(GOLD, "pixels_px.npz"))
    n, steps, seed, ml = (int(g[k]) for k in ("n", "steps", "seed", "max_len"))
    na = O.TIERS[tier]["NA"]
    for px in g["px"]:
        b = O.OracleBatch(tier, n, seed, max_episode_length=ml)
        want = g[f"{tier}_{int(px)}"]
        assert digest(b.state.render_pixels(int(px))) == int(want[0]), f"{px} px reset"
        for k in range(steps):
            b.step(O.random_actions(seed, k, n, na))
            assert digest(b.state.render_pixels(int(px))) == int(want[k + 1]), f"{px} px step {k}"
