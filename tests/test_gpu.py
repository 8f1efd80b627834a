"""GPU parity and API tests (run on a B200: pytest -m gpu).

Parity: the CUDA path (through the C ABI) against the C oracle -- which
tests/test_oracle_golden.py pins to the numpy reference -- on the same
seeded inputs: every SimState field, reward, done, newly-unlocked flags,
info, symbolic observations and pixel frames, bit for bit, including the
auto-reset pool, reset-stress runs and scrambled states that reach the
rare branches (enchanting, potions, ladders, boss waves, projectiles).
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _shapes(O, tier, n):
    return O.field_shapes(tier, n)


def _cmp_state(O, gb, ob_state, tier, n, skip=()):
    ex = gb.export_state(_shapes(O, tier, n))
    ox = ob_state.export_fields()
    bad = [f for f in O.FIELD_NAMES if f not in skip and not np.array_equal(ex[f], ox[f])]
    assert not bad, f"state fields differ: {bad}"


def _step_both(torch, gb, ob, a):
    obs, rew, done, newly, tm, fl = gb.step(torch.from_numpy(a).cuda())
    r2, d2, nw2, info = ob.step(a)
    assert np.array_equal(rew.cpu().numpy(), r2.astype(np.float32))
    assert np.array_equal(done.cpu().numpy().astype(bool), d2)
    assert np.array_equal(newly.cpu().numpy().astype(bool), nw2)
    assert np.array_equal(tm.cpu().numpy().view(np.uint32), info["time"])
    assert np.array_equal(fl.cpu().numpy(), info["floor"])
    return obs


@pytest.mark.parametrize("tier,n", [("classic", 512), ("extended", 384)])
def test_batch_reset_matches_oracle(torch_cuda, oracle_lib, tier, n):
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    gb = GridrogueBatch(n, tier, 11, "symbolic")
    obs = gb.reset().cpu().numpy()
    ob = O.OracleBatch(tier, n, 11, threads=8)
    _cmp_state(O, gb, ob.state, tier, n)
    assert np.array_equal(obs, ob.state.encode_symbolic())
    assert np.array_equal(gb.level_seeds(), ob.state.export_fields()["params_seed"])


@pytest.mark.parametrize("tier,n,steps,seed,max_len", [
    ("classic", 256, 300, 0, None),
    ("extended", 256, 300, 0, None),
    ("extended", 128, 120, 3, 16),     # reset stress: every env resets every 16 steps
    ("classic", 128, 120, 4, 16),
    ("extended", 200, 150, 9, 40),
])
def test_rollout_parity(torch_cuda, oracle_lib, tier, n, steps, seed, max_len):
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    torch = torch_cuda
    gb = GridrogueBatch(n, tier, seed, "symbolic", max_len)
    gb.reset()
    ob = O.OracleBatch(tier, n, seed, max_episode_length=max_len, threads=8)
    na = O.TIERS[tier]["NA"]
    for k in range(steps):
        obs = _step_both(torch, gb, ob, O.random_actions(seed, k, n, na))
        assert np.array_equal(obs.cpu().numpy(), ob.state.encode_symbolic()), f"obs step {k}"
        if k % 25 == 0:
            _cmp_state(O, gb, ob.state, tier, n)
    _cmp_state(O, gb, ob.state, tier, n)
    s1, s2 = gb.stats(), ob.stats()
    assert s1["episodes"] == s2["episodes"] > 0
    assert s1["total_steps"] == s2["total_steps"]
    assert np.array_equal(s1["ach_episodes"], s2["ach_episodes"])
    assert abs(s1["total_return"] - s2["total_return"]) <= 1e-9 * max(1.0, abs(s2["total_return"]))


@pytest.mark.parametrize("tier,n,px,steps", [("classic", 64, 7, 60), ("extended", 64, 10, 60),
                                             ("classic", 32, 16, 20), ("extended", 16, 16, 20),
                                             ("classic", 24, 10, 20), ("extended", 24, 7, 20)])
def test_pixel_parity(torch_cuda, oracle_lib, tier, n, px, steps):
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    gb = GridrogueBatch(n, tier, 5, "pixels", 30, tile_px=px)
    obs = gb.reset().cpu().numpy()
    ob = O.OracleBatch(tier, n, 5, max_episode_length=30)
    assert np.array_equal(obs, ob.state.render_pixels(px))
    for k in range(steps):
        obs = _step_both(torch_cuda, gb, ob, O.random_actions(5, k, n, O.TIERS[tier]["NA"]))
        assert np.array_equal(obs.cpu().numpy(), ob.state.render_pixels(px)), f"pixels step {k}"


@pytest.mark.parametrize("tier", ["classic", "extended"])
def test_scrambled_state_parity(torch_cuda, oracle_lib, tier):
    """Rare branches: import the scrambled states of the fuzz golden into both
    sides and step them under batch semantics with the golden's actions."""
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    g = np.load(os.path.join(GOLD, f"fuzz_{tier}.npz"))
    n = int(g["n"])
    start = {f: g[f"start_{f}"] for f in O.FIELD_NAMES}
    gb = GridrogueBatch(n, tier, 21, "symbolic")
    gb.reset()
    gb.import_state(start)
    ob = O.OracleBatch(tier, n, 21)
    ob.state.import_fields(start)
    assert np.array_equal(gb.observe().cpu().numpy(), ob.state.encode_symbolic())
    for k, a in enumerate(g["actions"]):
        obs = _step_both(torch_cuda, gb, ob, a)
        assert np.array_equal(obs.cpu().numpy(), ob.state.encode_symbolic()), f"obs step {k}"
        _cmp_state(O, gb, ob.state, tier, n)


def test_full_size_north_star_parity(torch_cuda):
    """The bench workload (65,536 extended envs, seed 0) against digests minted
    from the unmodified numpy reference (tests/golden/make_long_golden.py):
    the reset state (maps included) and observation, then 12 steps of reward /
    done / newly / info / observation / full state, the final per-field digests,
    the f64 episode accumulators and the level seeds."""
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200.layout import field_shapes, FIELD_NAMES
    from tests._digest import digest, state_digest
    torch = torch_cuda
    g = np.load(os.path.join(GOLD, "north_star_ext_n65536.npz"))
    n, seed, steps = int(g["n"]), int(g["seed"]), int(g["steps"])
    shapes = field_shapes("extended", n)
    gb = GridrogueBatch(n, "extended", seed, "symbolic")
    obs = gb.reset()
    assert state_digest(gb.export_state(shapes), FIELD_NAMES) == int(g["reset"][0]), "reset state"
    assert digest(obs.cpu().numpy()) == int(g["reset"][1]), "reset obs"
    for k in range(steps):
        obs, rew, done, newly, tm, fl = gb.step(gb.random_actions(seed, k))
        assert digest(rew.cpu().numpy()) == int(g["reward"][k]), f"reward step {k}"
        assert digest(done.cpu().numpy().astype(bool)) == int(g["done"][k]), f"done step {k}"
        assert digest(newly.cpu().numpy().astype(bool)) == int(g["newly"][k]), f"newly step {k}"
        assert digest(tm.cpu().numpy().view(np.uint32), fl.cpu().numpy()) == int(g["info"][k]), f"info step {k}"
        assert digest(obs.cpu().numpy()) == int(g["obs"][k]), f"obs step {k}"
        assert state_digest(gb.export_state(shapes), FIELD_NAMES) == int(g["state"][k]), f"state step {k}"
    ex = gb.export_state(shapes)
    bad = [f for f, dg in zip(FIELD_NAMES, g["final_fields"]) if digest(ex[f]) != int(dg)]
    assert not bad, f"fields differ from the reference: {bad}"
    assert digest(*gb.episode_progress()) == int(g["episode_acc"])
    assert digest(gb.level_seeds()) == int(g["level_seeds_digest"])
    assert gb.stats()["episodes"] == int(g["episodes"])


def test_batchenv_contract(torch_cuda, oracle_lib):
    """gridrogue_gym.BatchEnv semantics (bindings/tests/test_bindings.py)."""
    from paper_2402_16801_b200 import BatchEnv
    O = oracle_lib
    env = BatchEnv(4, tier="extended", seed=1)
    obs = env.reset()
    assert obs.shape == (4, 8268) and obs.dtype == np.float32
    obs, reward, done, info = env.step(np.zeros(4, np.int64))
    assert obs.shape == (4, 8268) and reward.dtype == np.float32 and reward.shape == (4,)
    assert done.shape == (4,) and done.dtype == bool
    assert info["newly_unlocked"].shape == (4, 67)
    assert BatchEnv(3, tier="classic", seed=1).reset().shape == (3, 1345)
    env = BatchEnv(4, tier="classic", seed=0)
    env.reset()
    with pytest.raises(ValueError, match="env 2"):
        env.step(np.array([0, 1, 99, 3]))
    with pytest.raises(ValueError, match="shape"):
        env.step(np.zeros(5, np.int64))
    with pytest.raises(RuntimeError, match="reset"):
        BatchEnv(2, tier="classic").step(np.zeros(2, np.int64))
    with pytest.raises(ValueError):
        BatchEnv(2, tier="classic", obs_mode="rgb")
    # bit parity of the host path with the oracle batch over 300 steps
    n = 20
    env = BatchEnv(n, tier="classic", seed=9)
    ob = O.OracleBatch("classic", n, 9)
    assert np.array_equal(env.reset(), ob.state.encode_symbolic())
    rng = np.random.default_rng(4)
    for _ in range(300):
        acts = rng.integers(0, 17, size=n)
        o1, r1, d1, i1 = env.step(acts)
        r2, d2, nw2, i2 = ob.step(acts)
        assert np.array_equal(r1, r2.astype(np.float32)) and np.array_equal(d1, d2)
        assert np.array_equal(o1, ob.state.encode_symbolic())
        assert np.array_equal(i1["newly_unlocked"], nw2) and np.array_equal(i1["time"], i2["time"])
    assert i1["episodes_completed"] == ob.stats()["episodes"]


def test_auto_reset_consumes_done(torch_cuda, oracle_lib):
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    gb = GridrogueBatch(4, "classic", 2, "symbolic")
    gb.reset()
    health = gb.export_field("health").view(np.float32).copy()
    health[1] = 0.0
    gb.import_field("health", health)
    _, _, done, *_ = gb.step(torch_cuda.zeros(4, dtype=torch_cuda.int64, device="cuda"))
    assert bool(done[1]) and not bool(done[0])
    assert not gb.export_field("done").any()
    assert gb.export_field("time").view(np.uint32)[1] == 0


def test_device_validation_and_policy(torch_cuda, oracle_lib):
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200.policies import RandomPolicy
    torch = torch_cuda
    gb = GridrogueBatch(1000, "extended", 3, "none")
    gb.reset()
    a = gb.random_actions(77, 5).cpu().numpy()
    assert np.array_equal(a, RandomPolicy(77, 43).actions_at(5, 1000))
    before = gb.export_field("time").copy()
    bad = torch.zeros(1000, dtype=torch.int64, device="cuda")
    bad[321] = 43
    with pytest.raises(ValueError, match="env 321"):
        gb.step(bad)
    assert np.array_equal(before, gb.export_field("time"))   # nothing mutated


def test_gymnax_facade(torch_cuda):
    from paper_2402_16801_b200 import make_craftax_env_from_name, EnvParams
    torch = torch_cuda
    env = make_craftax_env_from_name("Craftax-Symbolic-v1")
    params = EnvParams(n_envs=64)
    obs, state = env.reset(0, params)
    assert tuple(obs.shape) == (64, 8268)
    action = torch.zeros(64, dtype=torch.int64, device="cuda")
    obs, state, reward, done, info = env.step(1, state, action, params)
    assert tuple(reward.shape) == (64,) and done.dtype == torch.bool
    env = make_craftax_env_from_name("Craftax-Classic-Pixels-v1")
    obs, state = env.reset(3, EnvParams(n_envs=8))
    assert tuple(obs.shape) == (8, 63, 63, 3) and obs.dtype == torch.uint8


def test_sharded_batch_world_one(torch_cuda, oracle_lib):
    """ShardedBatch's exchange path (single rank) equals the plain step."""
    import torch.distributed as dist
    from paper_2402_16801_b200 import ShardedBatch
    O = oracle_lib
    torch = torch_cuda
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sb = ShardedBatch(96, "extended", 13, "symbolic", max_episode_length=20)
        sb.reset()
        ob = O.OracleBatch("extended", 96, 13, max_episode_length=20)
        for k in range(50):
            a = O.random_actions(13, k, 96, 43)
            obs, rew, done, *_ = sb.step(torch.from_numpy(a).cuda())
            r2, d2, _, _ = ob.step(a)
            assert np.array_equal(rew.cpu().numpy(), r2.astype(np.float32))
            assert np.array_equal(obs.cpu().numpy(), ob.state.encode_symbolic())
        assert sb.stats()["episodes"] == ob.stats()["episodes"]
    finally:
        dist.destroy_process_group()


def _golden_rollouts():
    with open(os.path.join(os.path.dirname(__file__), "golden", "bench_rollout_report.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", range(4))
def test_rollout_report_matches_reference(torch_cuda, case):
    """bench_report.run_rollout_report == the reference's run_rollout_report (bench.py:67-107)."""
    from paper_2402_16801_b200.bench_report import run_rollout_report
    g = _golden_rollouts()[case]
    tier, n, total, seed = g["args"]
    ref = g["report"]
    rep = run_rollout_report(tier, n, total, policy="random", seed=seed)
    for k in ("tier", "policy", "seed", "n_envs", "total_steps", "episodes_completed", "episodes_counted",
              "max_return", "achievement_rates"):
        assert rep[k] == ref[k], k
    # EpisodeStats.total_return is summed in a different order on the device
    assert rep["mean_return"] == pytest.approx(ref["mean_return"], abs=2e-6)
    assert rep["return_pct_of_max"] == pytest.approx(ref["return_pct_of_max"], abs=2e-4)


def test_speed_sweep_rows(torch_cuda):
    from paper_2402_16801_b200.bench_report import run_speed_sweep
    rows = run_speed_sweep("classic", [1, 64], 640)
    assert [r["workers"] for r in rows] == [1, 64]
    assert sum(r["best"] for r in rows) == 1
    assert all(r["sps"] > 0 for r in rows)
    assert rows[1]["steps"] == 640


def test_episode_progress_roundtrip(torch_cuda, oracle_lib):
    """BatchState.ep_return / ep_length / step_index export == the oracle's, and import restores them."""
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    n = 48
    gb = GridrogueBatch(n, "classic", 3, "none", 25)
    gb.reset()
    ob = O.OracleBatch("classic", n, 3, max_episode_length=25)
    for k in range(40):
        a = O.random_actions(3, k, n, O.TIERS["classic"]["NA"])
        gb.step(torch_cuda.from_numpy(a).cuda())
        ob.step(a)
    ret, length = gb.episode_progress()
    oret, olen = ob.episode_progress()
    assert np.array_equal(length, olen)
    assert np.array_equal(ret, oret)
    assert gb.step_index == 40
    gb.set_episode_progress(ret * 0 + 1.5, length + 1)
    r2, l2 = gb.episode_progress()
    assert np.all(r2 == 1.5) and np.array_equal(l2, length + 1)


@pytest.mark.parametrize("name", ["game_state_classic.bin", "game_state_extended.bin",
                                  "game_state_classic_batch.bin", "game_state_extended_batch.bin"])
def test_game_state_blob_roundtrip(torch_cuda, name):
    """A blob written by the reference's serializer loads into a device batch and writes back identically."""
    from paper_2402_16801_b200 import serialize as S
    with open(os.path.join(os.path.dirname(__file__), "golden", name), "rb") as fh:
        blob = fh.read()
    meta, data = S._unpack(blob, "game_state")
    gb = S.state_from_bytes(blob, obs_mode="symbolic")
    out = gb.export_state()
    for f, a in out.items():
        assert np.array_equal(a, data[f]), f
    meta2, data2 = S._unpack(S.state_to_bytes(gb), "game_state")
    assert meta2 == meta
    for f in out:
        assert np.array_equal(data2[f], data[f]), f
    doc = S.state_to_json(gb)
    gb2 = S.state_from_json(json.loads(json.dumps(doc)), obs_mode="none")
    for f, a in gb2.export_state().items():
        assert np.array_equal(a, data[f]), f
    # the loaded batch renders and steps
    obs = gb.observe()
    assert obs.shape[0] == gb.n
    gb.set_validate(False)
    gb.random_actions(1, 0)
    gb.step(gb.actions)


@pytest.mark.parametrize("tier", ["classic", "extended"])
def test_batch_checkpoint_resume_is_exact(torch_cuda, tier):
    """batch_to_bytes at step 20, resumed in a new batch: 25 more steps equal the uninterrupted run."""
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200 import serialize as S
    n = 96
    a = GridrogueBatch(n, tier, 21, "symbolic", 12)   # short episodes: resets inside the window
    a.reset()
    a.set_validate(False)
    for t in range(20):
        a.random_actions(4, t)
        a.step(a.actions)
    blob = S.batch_to_bytes(a)
    b = S.batch_from_bytes(blob, obs_mode="symbolic")
    b.set_validate(False)
    assert b.step_index == a.step_index == 20
    for t in range(20, 45):
        a.random_actions(4, t)
        oa = a.step(a.actions)[0].clone()
        b.random_actions(4, t)
        ob = b.step(b.actions)[0]
        assert torch_cuda.equal(oa, ob), f"obs step {t}"
    sa, sb = a.export_state(), b.export_state()
    for f in sa:
        assert np.array_equal(sa[f], sb[f]), f
    xa, xb = a.stats(), b.stats()
    assert xa["episodes"] == xb["episodes"] > 0 and xa["total_steps"] == xb["total_steps"]
    assert np.array_equal(xa["ach_episodes"], xb["ach_episodes"])
    assert xa["total_return"] == pytest.approx(xb["total_return"], rel=1e-12)
    ra, la = a.episode_progress()
    rb, lb = b.episode_progress()
    assert np.array_equal(la, lb) and np.array_equal(ra, rb)


def _ued():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "ued_levels.npz"))


@pytest.mark.parametrize("tag", ["classic_3", "classic_1001", "extended_5", "extended_77", "extended_2024"])
def test_ued_levels_match_reference(torch_cuda, tag):
    """make_level_params -> mutate_noise -> generate_world -> mutate_swap / mutate_rswap
    -> install_world on the device equal the reference (tests/golden/make_mutate_golden.py)."""
    from paper_2402_16801_b200 import GridrogueBatch, rng
    from paper_2402_16801_b200.levels import LevelBuffer
    from paper_2402_16801_b200.layout import field_shapes
    g = _ued()
    tier, seed = tag.split("_")[0], int(tag.split("_")[1])
    gb = GridrogueBatch(4, tier, 0, "symbolic")
    gb.reset()
    lv = LevelBuffer(gb, 3)
    lv.set_params(0, [seed, seed, seed])
    s, a, f = lv.params(0, 3)
    assert np.array_equal(a[0].view(np.uint32), g[f"{tag}_params_angles"].view(np.uint32))
    assert np.array_equal(f[0], g[f"{tag}_params_floor_seeds"])
    lv.mutate("noise", [0, 1, 2], [rng.make_stream(seed + 1)] * 3)
    s, a, f = lv.params(0, 3)
    for k in range(3):
        assert np.array_equal(a[k].view(np.uint32), g[f"{tag}_noisy_angles"].view(np.uint32))
        assert np.array_equal(f[k], g[f"{tag}_noisy_floor_seeds"]) and s[k] == g[f"{tag}_noisy_seed"]
    lv.generate(0, 3)

    def same_world(w, pre):
        assert np.array_equal(w["blocks"], g[f"{pre}_blocks"])
        assert np.array_equal(w["items"], g[f"{pre}_items"])
        assert np.array_equal(w["spawn"], g[f"{pre}_spawn"])
        assert np.array_equal(w["ladders"], g[f"{pre}_ladders"])
        assert np.array_equal(w["chests"], g[f"{pre}_chests"])
        assert np.array_equal(w["potion"], g[f"{pre}_potion"])

    same_world(lv.world(0), f"{tag}_world")
    lv.mutate("swap", [1], [rng.make_stream(seed + 2)])
    same_world(lv.world(1), f"{tag}_swap")
    lv.mutate("rswap", [2], [rng.make_stream(seed + 3)])
    same_world(lv.world(2), f"{tag}_rswap")
    key = int(g[f"{tag}_install_key"])
    assert key == rng.split(rng.make_stream(seed + 4), 0).key
    lv.install([2], [2], [key])
    st = gb.export_state()
    for name, (dt, shape) in field_shapes(tier, 1).items():
        assert np.array_equal(st[name][2:3], g[f"{tag}_state_{name}"]), name
    # the installed env steps and renders like any other
    gb.set_validate(False)
    gb.random_actions(0, 0)
    gb.step(gb.actions)


def test_ppo_short_run(torch_cuda):
    """A short PPO run on the device engine: finite losses, episodes complete, throughput reported."""
    from paper_2402_16801_b200.ppo import PPOConfig, train
    cfg = PPOConfig(tier="classic", n_envs=256, n_steps=32, total_timesteps=256 * 32 * 6)
    res = train(cfg, log=lambda s: None)
    assert res["updates"] == 6 and res["env_steps"] == 256 * 32 * 6
    assert res["sps"] > 0
    for row in res["history"]:
        assert all(np.isfinite([row["loss"], row["pg_loss"], row["v_loss"], row["entropy"]]))


def _two_rank_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle as O
        from paper_2402_16801_b200 import ShardedBatch
        n = 96
        sb = ShardedBatch(n, "extended", 17, "symbolic", max_episode_length=15)
        sb.reset()
        ob = O.OracleBatch("extended", n, 17, max_episode_length=15)
        lo, hi = sb.lo, sb.hi
        for k in range(40):
            a = O.random_actions(17, k, n, 43)
            obs, rew, done, *_ = sb.step(torch.from_numpy(a[lo:hi]).cuda())
            r2, d2, _, _ = ob.step(a)
            assert np.array_equal(rew.cpu().numpy(), r2[lo:hi].astype(np.float32)), f"reward step {k}"
            assert np.array_equal(done.cpu().numpy().astype(bool), d2[lo:hi]), f"done step {k}"
            assert np.array_equal(obs.cpu().numpy(), ob.state.encode_symbolic()[lo:hi]), f"obs step {k}"
        st = sb.stats()
        assert st["episodes"] == ob.stats()["episodes"] > 0
        seeds = sb.batch.export_state()["params_seed"]
        assert np.array_equal(seeds, ob.state.export_fields()["params_seed"][lo:hi])
        q.put((rank, "ok"))
        dist.destroy_process_group()
    except Exception as ex:   # reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_sharded_batch_two_ranks_one_gpu(torch_cuda):
    """Two ranks (two processes, gloo exchange) on one GPU: each shard equals the
    matching slice of one global batch -- pool slots by global done rank, the
    batch-wide flags, per-rank worldgen of the consumed slots."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 200)
    ps = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"


LONG = sorted(f[len("long_"):-4] for f in os.listdir(GOLD) if f.startswith("long_"))


@pytest.mark.parametrize("name", LONG)
def test_long_rollout_parity_10k(torch_cuda, name):
    """BASELINE.json north star, pinned to the reference itself: 10^4-step random
    rollouts of all four variants (Classic/Full x Symbolic/Pixels), and of the
    symbolic variants at 1,024 envs with natural episode ends, against digests
    minted from the unmodified numpy reference (tests/golden/make_long_golden.py):
    every step's reward / done / observation, the full SimState (maps included)
    and the f64 episode accumulators every 2,500 steps, final fields and
    EpisodeStats.  Episodes are capped at 700 steps, so every env lives through
    many auto-resets."""
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200.layout import field_shapes, FIELD_NAMES
    from tests._digest import digest, state_digest
    torch = torch_cuda
    g = np.load(os.path.join(GOLD, f"long_{name}.npz"))
    tier, obs_mode, n = str(g["tier"]), str(g["obs_mode"]), int(g["n"])
    steps, seed, ml, every, px = (int(g[k]) for k in ("steps", "seed", "max_len", "every", "tile_px"))
    obs_every = int(g["obs_every"]) if "obs_every" in g.files else 1
    shapes = field_shapes(tier, n)
    gb = GridrogueBatch(n, tier, seed, obs_mode, ml or None, tile_px=px, newly=False, info=False)
    obs = gb.reset()
    assert state_digest(gb.export_state(shapes), FIELD_NAMES) == int(g["reset"][0]), "reset state"
    assert digest(obs.cpu().numpy()) == int(g["reset"][1]), "reset obs"
    gb.set_validate(False)
    c = 0
    for k in range(steps):
        obs, rew, done, *_ = gb.step(gb.random_actions(seed, k))
        assert digest(rew.cpu().numpy()) == int(g["reward"][k]), f"reward step {k}"
        assert digest(done.cpu().numpy().astype(bool)) == int(g["done"][k]), f"done step {k}"
        if k % obs_every == 0:
            assert digest(obs.cpu().numpy()) == int(g["obs"][k]), f"obs step {k}"
        if (k + 1) % every == 0:
            assert state_digest(gb.export_state(shapes), FIELD_NAMES) == int(g["ckpt"][c][0]), f"state step {k}"
            assert digest(*gb.episode_progress()) == int(g["ckpt"][c][1]), f"episode acc step {k}"
            c += 1
    ex = gb.export_state(shapes)
    bad = [f for f, dg in zip(FIELD_NAMES, g["final_fields"]) if digest(ex[f]) != int(dg)]
    assert not bad, f"fields differ from the reference: {bad}"
    s = gb.stats()
    assert s["episodes"] == int(g["episodes"]) >= (n * (steps // ml) if ml else n)
    assert s["total_steps"] == int(g["total_steps"])
    assert np.array_equal(s["ach_episodes"], g["ach_episodes"])
    assert np.array_equal(gb.level_seeds(), g["level_seeds"])


def test_batchenv_determinism_and_no_allocation_growth(torch_cuda):
    """bindings/tests/test_bindings.py: two envs with one seed agree step for step;
    stepping allocates nothing per step (host: tracemalloc; device: the CUDA
    allocator and the library's captured step graphs)."""
    import tracemalloc
    from paper_2402_16801_b200 import BatchEnv
    a, b = BatchEnv(8, tier="classic", seed=5), BatchEnv(8, tier="classic", seed=5)
    a.reset(); b.reset()
    rng = np.random.default_rng(0)
    for _ in range(50):
        acts = rng.integers(0, 17, size=8)
        oa, ra, da, _ = a.step(acts)
        ob, rb, db, _ = b.step(acts)
        assert np.array_equal(ra, rb) and np.array_equal(da, db) and np.array_equal(oa, ob)
    env = BatchEnv(16, tier="classic", seed=3, obs_mode="none")
    env.reset()
    acts = np.zeros(16, np.int64)
    for _ in range(200):
        env.step(acts)
    torch_cuda.cuda.synchronize()
    dev0 = torch_cuda.cuda.memory_allocated()
    tracemalloc.start()
    s0 = tracemalloc.take_snapshot()
    for _ in range(400):
        env.step(acts)
    s1 = tracemalloc.take_snapshot()
    tracemalloc.stop()
    growth = sum(st.size_diff for st in s1.compare_to(s0, "filename") if st.size_diff > 0)
    assert growth < 2_000_000
    torch_cuda.cuda.synchronize()
    assert torch_cuda.cuda.memory_allocated() == dev0


@pytest.mark.parametrize("tier,obs_mode,n", [("classic", "symbolic", 1), ("extended", "symbolic", 1),
                                             ("extended", "pixels", 3), ("classic", "pixels", 1),
                                             ("extended", "symbolic", 129)])
def test_tiny_and_ragged_batches(torch_cuda, oracle_lib, tier, obs_mode, n):
    """Edge sizes: a single env, odd counts, one env past a 128-env block."""
    from paper_2402_16801_b200 import GridrogueBatch
    O = oracle_lib
    torch = torch_cuda
    gb = GridrogueBatch(n, tier, 44, obs_mode, 9)
    obs = gb.reset()
    ob = O.OracleBatch(tier, n, 44, max_episode_length=9)
    px = gb.tile_px
    ref = (lambda: ob.state.encode_symbolic()) if obs_mode == "symbolic" else (lambda: ob.state.render_pixels(px))
    assert np.array_equal(obs.cpu().numpy(), ref())
    for k in range(40):
        a = O.random_actions(44, k, n, O.TIERS[tier]["NA"])
        obs, rew, done, *_ = gb.step(torch.from_numpy(a).cuda())
        r2, d2, _, _ = ob.step(a)
        assert np.array_equal(rew.cpu().numpy(), r2.astype(np.float32)), f"reward step {k}"
        assert np.array_equal(obs.cpu().numpy(), ref()), f"obs step {k}"
    _cmp_state(O, gb, ob.state, tier, n)


@pytest.mark.parametrize("tier,n,max_len", [("extended", 1024, None), ("extended", 2048, 12), ("classic", 1024, 9)])
def test_small_batch_paths_match_plain_path(torch_cuda, monkeypatch, tier, n, max_len):
    """The small-batch step (speculative pool worldgen beside k_step, 512-thread
    extended worldgen) produces exactly what the plain step does: same rewards,
    dones, observations and final state, including steps where the done count
    outruns the speculation (max_episode_length: every env resets at once)."""
    import torch
    from paper_2402_16801_b200 import GridrogueBatch

    def run(spec, wide):
        monkeypatch.setenv("GR_SPEC", spec)
        monkeypatch.setenv("GR_WG_WIDE", wide)
        gb = GridrogueBatch(n, tier, 5, "symbolic", max_episode_length=max_len)
        gb.set_validate(False)
        obs0 = gb.reset().clone()
        out = [obs0]
        for t in range(40):
            gb.random_actions(5, t)
            obs, rew, done, *_ = gb.step(gb.actions)
            out += [obs.clone(), rew.clone(), done.clone()]
        st = gb.export_state()
        counters = gb.worldgen_counters()
        return out, st, counters

    a, sa, ca = run("1", "1")
    b, sb, cb = run("0", "0")
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    for k in sb:
        assert np.array_equal(sa[k], sb[k]), k
    assert ca["worlds"] >= cb["worlds"]   # the speculative pass may make a few unused worlds


@pytest.mark.parametrize("n_actions", [17, 43])
def test_fused_ppo_objective_matches_torch(torch_cuda, n_actions):
    """The fused PPO objective kernel (gr_ppo.cu) against a plain PyTorch fp32
    statement of the same loss: value and gradients (tolerance 1e-5 relative
    on the loss terms, 1e-6 absolute on the gradients)."""
    import torch
    from paper_2402_16801_b200.ppo import ppo_objective
    g = torch.Generator(device="cuda").manual_seed(n_actions)
    B = 8192
    z = torch.randn(B, n_actions, device="cuda", generator=g) * 2
    v = torch.randn(B, device="cuda", generator=g)
    act = torch.randint(0, n_actions, (B,), device="cuda", generator=g)
    logp_old = torch.log_softmax(z + 0.3 * torch.randn(B, n_actions, device="cuda", generator=g), -1).gather(
        -1, act[:, None]).squeeze(-1)
    adv = torch.randn(B, device="cuda", generator=g) * 3 + 0.5
    v_old = v + 0.3 * torch.randn(B, device="cuda", generator=g)
    ret = v + torch.randn(B, device="cuda", generator=g)
    eps, cv, ce = 0.2, 0.5, 0.01

    z1, v1 = z.clone().requires_grad_(), v.clone().requires_grad_()
    loss1, st = ppo_objective(z1, v1, act, logp_old, adv, v_old, ret, eps, cv, ce)
    loss1.backward()

    z2, v2 = z.clone().requires_grad_(), v.clone().requires_grad_()
    lp_all = torch.log_softmax(z2, -1)
    lp = lp_all.gather(-1, act[:, None]).squeeze(-1)
    ratio = torch.exp(lp - logp_old)
    a_ = (adv - adv.mean()) / (adv.std() + 1e-8)
    pg = -torch.min(ratio * a_, ratio.clamp(1 - eps, 1 + eps) * a_).mean()
    vc = v_old + (v2 - v_old).clamp(-eps, eps)
    vl = 0.5 * torch.max((v2 - ret) ** 2, (vc - ret) ** 2).mean()
    ent = -(lp_all.exp() * lp_all).sum(-1).mean()
    loss2 = pg + cv * vl - ce * ent
    loss2.backward()

    ref = torch.stack([loss2, pg, vl, ent]).detach()
    assert torch.allclose(st, ref, rtol=1e-5, atol=1e-6), (st, ref)
    assert torch.allclose(loss1.detach(), loss2.detach(), rtol=1e-5, atol=1e-6)
    assert torch.allclose(z1.grad, z2.grad, rtol=1e-4, atol=1e-6), (z1.grad - z2.grad).abs().max()
    assert torch.allclose(v1.grad, v2.grad, rtol=1e-4, atol=1e-6), (v1.grad - v2.grad).abs().max()


def _rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


@pytest.mark.parametrize("n_actions", [17, 43])
def test_manual_learner_matches_autograd(torch_cuda, n_actions):
    """learner.ManualLearner (bf16 forward on cuBLAS, grp_ppo_loss_bf16, the
    hand-written backward with grp_bias_grad) against autocast + autograd of
    the same module and the fused fp32 objective: forward outputs, loss terms
    and every parameter gradient (relative L2 error <= 2e-2: both run bf16
    GEMMs and bf16 activations, in different accumulation orders); the pad
    rows of the action head get exactly zero gradient."""
    import torch
    from paper_2402_16801_b200.learner import ManualLearner, pad_actions
    from paper_2402_16801_b200.ppo import make_fused_model, ppo_objective
    torch.manual_seed(n_actions)
    B, K, L = 2048, 8320, 512
    A = pad_actions(n_actions)
    model = make_fused_model(K, A, L).cuda()
    with torch.no_grad():
        model.actor[-1].weight[n_actions:].zero_()
        model.actor[-1].bias[n_actions:].zero_()
        for p in model.parameters():   # non-zero biases exercise the bias paths
            if p.dim() == 1:
                p.add_(0.05 * torch.randn_like(p))
        model.actor[-1].bias[n_actions:].zero_()
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.rand(B, K, device="cuda", generator=g) < 0.05).to(torch.bfloat16)
    x[:, 8268:] = 0
    act = torch.randint(0, n_actions, (B,), device="cuda", generator=g)
    logp_old = -torch.rand(B, device="cuda", generator=g) * 3 - 0.5
    adv = torch.randn(B, device="cuda", generator=g)
    v_old = torch.randn(B, device="cuda", generator=g) * 0.1
    ret = v_old + torch.randn(B, device="cuda", generator=g) * 0.5
    eps, cv, ce = 0.2, 0.5, 0.01

    # autograd reference on a copy of the module
    import copy
    ref = copy.deepcopy(model)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        zl, zv = ref(x)
    loss_r, st_r = ppo_objective(zl[:, :n_actions].float(), zv.float(), act, logp_old, adv, v_old, ret, eps, cv, ce)
    loss_r.backward()

    ln = ManualLearner(model, n_actions, B, torch.device("cuda"))
    logits, value = ln.forward(x)
    assert _rel(logits, zl) < 1e-2 and _rel(value.squeeze(-1), zv) < 1e-2
    st = torch.zeros(4, device="cuda")
    ln.loss(act, logp_old, adv, v_old, ret, eps, cv, ce, st)
    ln.backward(x)
    torch.cuda.synchronize()
    assert torch.allclose(st, st_r, rtol=2e-2, atol=1e-4), (st, st_r)
    for (name, p), pr in zip(model.named_parameters(), ref.parameters()):
        assert p.grad.shape == pr.grad.shape
        assert _rel(p.grad, pr.grad) < 2e-2, (name, _rel(p.grad, pr.grad))
    assert bool((model.actor[-1].weight.grad[n_actions:] == 0).all())
    assert bool((model.actor[-1].bias.grad[n_actions:] == 0).all())
    assert bool((ln.dlogits[:, n_actions:] == 0).all())


def test_bias_grad_kernel_exact(torch_cuda):
    """grp_bias_grad against a float64 statement: dz = bf16(dy (1 - y^2))
    bit for bit, db = column sums of dz (fp32 accumulation: 1e-5 relative),
    for the split two-source layout, an unaligned width (scalar path), and
    deterministic across calls."""
    import torch
    from paper_2402_16801_b200._lib import lib
    g = torch.Generator(device="cuda").manual_seed(5)
    for rows, cols, split in ((8192, 1024, 512), (777, 43, 43), (300, 1, 1)):
        y = torch.tanh(torch.randn(rows, cols, device="cuda", generator=g)).to(torch.bfloat16)
        da = torch.randn(rows, max(split, 1), device="cuda", generator=g).to(torch.bfloat16)
        db_ = torch.randn(rows, max(cols - split, 1), device="cuda", generator=g).to(torch.bfloat16)
        dy = torch.cat([da[:, :split], db_[:, :cols - split]], 1)
        dz = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda")
        out = [torch.empty(cols, device="cuda") for _ in range(2)]
        work = torch.zeros(32 * cols, device="cuda")
        ctr = torch.zeros((cols + 63) // 64, dtype=torch.int32, device="cuda")
        for o in out:
            rc = lib().grp_bias_grad(y.data_ptr(), y.stride(0), da.data_ptr(), da.stride(0), db_.data_ptr(),
                                     db_.stride(0), split, rows, cols, dz.data_ptr(), o.data_ptr(), work.data_ptr(),
                                     32, ctr.data_ptr(), 1, 0, 0, 0, torch.cuda.current_stream().cuda_stream)
            assert rc == 0
        torch.cuda.synchronize()
        ref_dz = (dy.float() * (1 - y.float() ** 2)).to(torch.bfloat16)
        assert torch.equal(dz, ref_dz), (rows, cols)
        ref_db = ref_dz.double().sum(0)
        assert torch.allclose(out[0].double(), ref_db, rtol=1e-5, atol=1e-4), (rows, cols)
        assert torch.equal(out[0], out[1])
        assert int(ctr.abs().sum()) == 0
    # batched: the actor / critic pair of a hidden layer, [2, rows, cols]
    rows, cols = 4096, 512
    y = torch.tanh(torch.randn(2, rows, cols, device="cuda", generator=g)).to(torch.bfloat16)
    dy = torch.randn(2, rows, cols, device="cuda", generator=g).to(torch.bfloat16)
    dz = torch.empty_like(dy)
    db = torch.empty(2, cols, device="cuda")
    work = torch.zeros(2 * 32 * cols, device="cuda")
    ctr = torch.zeros(2 * (cols // 64), dtype=torch.int32, device="cuda")
    rc = lib().grp_bias_grad(y.data_ptr(), cols, dy.data_ptr(), cols, None, 0, cols, rows, cols, dz.data_ptr(),
                             db.data_ptr(), work.data_ptr(), 32, ctr.data_ptr(), 2, rows * cols, rows * cols,
                             rows * cols, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert rc == 0
    ref_dz = (dy.float() * (1 - y.float() ** 2)).to(torch.bfloat16)
    assert torch.equal(dz, ref_dz)
    assert torch.allclose(db.double(), ref_dz.double().sum(1), rtol=1e-5, atol=1e-4)
    # grp_bias_tanh: z <- bf16(tanh(z + bias[b])) (float tanh: within 1 bf16 ulp of the float64 value)
    z = torch.randn(2, rows, cols, device="cuda", generator=g).to(torch.bfloat16)
    bias = torch.randn(2, cols, device="cuda", generator=g).to(torch.bfloat16)
    ref = torch.tanh(z.double() + bias.double()[:, None, :])
    assert lib().grp_bias_tanh(z.data_ptr(), bias.data_ptr(), 2, rows, cols,
                               torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert float((z.double() - ref).abs().max()) <= 2 ** -8


def test_rows_to_bf16_exact(torch_cuda):
    """grp_rows_to_bf16 (the rollout buffer's copy of a step's observation):
    equal to torch's float32 -> bf16 cast into the padded rows, pads untouched."""
    import torch
    from paper_2402_16801_b200._lib import lib
    g = torch.Generator(device="cuda").manual_seed(2)
    src = torch.randn(1000, 8268, device="cuda", generator=g) * 3
    dst = torch.full((1000, 8320), 7.0, dtype=torch.bfloat16, device="cuda")
    assert lib().grp_rows_to_bf16(src.data_ptr(), 1000, 8268, dst.data_ptr(), 8320,
                                  torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(dst[:, :8268], src.to(torch.bfloat16))
    assert bool((dst[:, 8268:] == 7.0).all())
    src = torch.randn(300, 1345, device="cuda", generator=g)   # Craftax-Classic rows: the scalar path
    dst = torch.full((300, 1408), 7.0, dtype=torch.bfloat16, device="cuda")
    assert lib().grp_rows_to_bf16(src.data_ptr(), 300, 1345, dst.data_ptr(), 1408,
                                  torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(dst[:, :1345], src.to(torch.bfloat16))
    assert bool((dst[:, 1345:] == 7.0).all())


def test_clip_adam_matches_torch(torch_cuda):
    """grp_clip_adam (global-norm clip of the scaled gradient + Adam + the
    bf16 copy) against torch.nn.utils.clip_grad_norm_ and torch.optim.Adam
    (capturable, fused) over 5 steps, once with a clipping norm and once
    without: parameters within 2e-6 relative, the bf16 copy equal to
    bf16(params)."""
    import torch
    from paper_2402_16801_b200._lib import lib
    g = torch.Generator(device="cuda").manual_seed(9)
    n = 1_000_003
    for max_norm, scale in ((0.5, 0.5), (1e9, 1.0)):
        p0 = torch.randn(n + 5, device="cuda", generator=g)[:n].clone()
        grads = [torch.randn(n, device="cuda", generator=g) * 1e-3 for _ in range(5)]
        pr = torch.nn.Parameter(p0.clone())
        lr = torch.tensor(3e-4, device="cuda")
        opt = torch.optim.Adam([pr], lr=lr, eps=1e-5, capturable=True, fused=True)
        P, M, V = p0.clone(), torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
        Pb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        step = torch.zeros(1, device="cuda")
        work = torch.zeros(300, device="cuda")
        ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
        for gr in grads:
            pr.grad = gr * scale
            torch.nn.utils.clip_grad_norm_([pr], max_norm)
            opt.step()
            rc = lib().grp_clip_adam(P.data_ptr(), gr.data_ptr(), M.data_ptr(), V.data_ptr(), Pb.data_ptr(), n,
                                     lr.data_ptr(), step.data_ptr(), 0.9, 0.999, 1e-5, scale, max_norm,
                                     work.data_ptr(), ctr.data_ptr(), torch.cuda.current_stream().cuda_stream)
            assert rc == 0
        torch.cuda.synchronize()
        assert float(step) == 5.0
        assert _rel(P - p0, pr.detach() - p0) < 2e-3, _rel(P - p0, pr.detach() - p0)
        assert torch.allclose(P, pr.detach(), rtol=2e-6, atol=1e-7)
        assert torch.equal(Pb, P.to(torch.bfloat16))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fused_sampler_distribution(torch_cuda, dtype):
    """grp_sample_actions: actions follow softmax(logits) (empirical
    frequencies within 5 sigma over 65,536 draws), log p(a) equals the torch
    log-softmax, values and the previous reward / done are copied."""
    import torch
    from paper_2402_16801_b200._lib import lib
    n, A = 65536, 43
    g = torch.Generator(device="cuda").manual_seed(3)
    row = torch.randn(A, device="cuda", generator=g) * 1.5
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    z = row.to(dt).expand(n, A).contiguous()
    v = torch.randn(n, 1, device="cuda", generator=g).to(dt)
    ctr = torch.tensor([7], dtype=torch.int64, device="cuda")
    a1 = torch.empty(n, dtype=torch.int64, device="cuda")
    a2 = torch.empty_like(a1)
    lp = torch.empty(n, device="cuda")
    vo = torch.empty(n, device="cuda")
    pr = torch.randn(n, device="cuda", generator=g)
    pd = (torch.rand(n, device="cuda", generator=g) < 0.3).to(torch.uint8)
    ro, do = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    rc = lib().grp_sample_actions(z.data_ptr(), v.data_ptr(), 1 if dtype == "bf16" else 0, n, A, A, 1, 12345,
                                  ctr.data_ptr(), 5, a1.data_ptr(), a2.data_ptr(), lp.data_ptr(), vo.data_ptr(),
                                  pr.data_ptr(), pd.data_ptr(), ro.data_ptr(), do.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert rc == 0
    assert torch.equal(a1, a2) and int(a1.min()) >= 0 and int(a1.max()) < A
    p = torch.softmax(z[0].float(), -1)
    freq = torch.bincount(a1, minlength=A).float() / n
    sigma = torch.sqrt(p * (1 - p) / n)
    assert bool(((freq - p).abs() <= 5 * sigma + 1e-4).all()), (freq - p).abs().max()
    ref_lp = torch.log_softmax(z.float(), -1).gather(-1, a1[:, None]).squeeze(-1)
    assert torch.allclose(lp, ref_lp, rtol=1e-5, atol=1e-6)
    assert torch.equal(vo, v.float().squeeze(-1))
    assert torch.equal(ro, pr) and torch.equal(do, pd.float())


def _ppo_two_rank_worker(rank, world, port, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                          LOCAL_RANK="0")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2402_16801_b200.ppo import PPOConfig, train
        cfg = PPOConfig(tier="classic", n_envs=128, n_steps=16, total_timesteps=128 * 2 * 16 * 4)
        res = train(cfg, log=lambda s: None)
        q.put((rank, "ok", res["param_checksum"], res["updates"], res["env_steps"],
               [r["loss"] for r in res["history"]]))
        dist.destroy_process_group()
    except Exception:   # reported to the parent
        import traceback
        q.put((rank, traceback.format_exc(), None, None, None, None))


def test_graphed_ppo_two_ranks_one_gpu(torch_cuda):
    """The graphed learner with two ranks (two processes sharing the GPU, gloo
    all-reduce of the flat gradient): the ranks' shards differ, their
    averaged updates must leave identical weights on both ranks."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + (os.getpid() % 150)
    ps = [ctx.Process(target=_ppo_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=900) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, msg, *_ in res:
        assert msg == "ok", f"rank {rank}: {msg}"
    (_, _, c0, u0, s0, l0), (_, _, c1, u1, s1, l1) = res
    assert u0 == u1 == 4 and s0 == s1 == 128 * 2 * 16 * 4
    assert c0 == c1, (c0, c1)
    assert all(np.isfinite(l0)) and all(np.isfinite(l1))


def test_batchenv_returned_obs_are_never_overwritten(torch_cuda):
    """BatchEnv hands out observations without a per-step copy (two pinned
    buffers, reused only when the caller holds no reference): arrays the
    caller keeps stay as returned, like the reference's fresh arrays."""
    from paper_2402_16801_b200 import BatchEnv
    env = BatchEnv(6, tier="extended", seed=2)
    kept = [env.reset()]
    snap = [kept[0].copy()]
    acts = np.zeros(6, np.int64)
    for k in range(6):
        o, *_ = env.step(acts + (k % 5))
        kept.append(o)
        snap.append(o.copy())
    for a, b in zip(kept, snap):
        assert np.array_equal(a, b)
    # a loop that drops each observation reuses the two buffers (no copies)
    ids = set()
    for k in range(8):
        o, *_ = env.step(acts)
        ids.add(o.__array_interface__["data"][0])
        del o
    assert len(ids) <= 2


@pytest.mark.parametrize("tier,n_act", [("extended", 43), ("classic", 17)])
def test_batchenv_delta_obs_transfer_matches_oracle(torch_cuda, tier, n_act):
    """BatchEnv(obs_transfer="delta") -- gr_host_obs_attach'ed pinned buffers
    that receive only the words changed since their last observation --
    returns the same arrays as the oracle (bindings/src/gridrogue_gym/
    __init__.py:63-95) under reset stress, while the caller holds some
    returned arrays (buffer rotation and the copy fallback) and drops others
    (buffer reuse)."""
    import oracle as O
    from paper_2402_16801_b200 import BatchEnv
    n, seed, max_len = 48, 11, 12
    env = BatchEnv(n, tier=tier, seed=seed, max_episode_length=max_len, obs_transfer="delta")
    ob = O.OracleBatch(tier, n, seed, max_episode_length=max_len)
    obs = env.reset()
    assert not obs.flags.writeable
    with pytest.raises(ValueError):
        obs.flags.writeable = True
    assert np.array_equal(obs, ob.state.encode_symbolic())
    held = []
    rng = np.random.default_rng(4)
    for k in range(60):
        a = rng.integers(0, n_act, size=n)
        obs, rew, done, _ = env.step(a)
        r2, d2, _, _ = ob.step(a)
        want = ob.state.encode_symbolic()
        assert np.array_equal(obs.view(np.uint32), want.view(np.uint32)), f"obs differs at step {k}"
        assert np.array_equal(rew, r2.astype(np.float32)) and np.array_equal(done, d2)
        if k % 7 == 3:
            held.append((obs, want))     # keep this buffer out of the rotation for a while
        if k % 7 == 6:
            held.clear()
    for o, w in held:                     # held arrays were never overwritten
        assert np.array_equal(o, w)
    obs = env.reset()                     # a reset through an attached buffer
    ob = O.OracleBatch(tier, n, seed, max_episode_length=max_len)
    assert np.array_equal(obs, ob.state.encode_symbolic())
    with pytest.raises(ValueError):
        BatchEnv(2, tier=tier, obs_mode="pixels", obs_transfer="delta")


def test_host_obs_delta_list_growth(torch_cuda):
    """The changed-word list outgrows its first capacity (every word of a
    fresh reset differs from a zeroed buffer when the capacity is tiny
    relative to the row): several passes, same result as a dense copy."""
    import ctypes
    from paper_2402_16801_b200 import _lib, GridrogueBatch
    import oracle as O
    n = 64
    gb = GridrogueBatch(n, "extended", 2, "symbolic", device=0)
    h = torch_cuda.zeros((n, 8268), dtype=torch_cuda.float32, pin_memory=True)
    p = ctypes.c_void_p(h.data_ptr())
    _lib.check(_lib.lib().gr_host_obs_attach(gb.h, p))
    _lib.check(_lib.lib().gr_reset_host(gb.h, p))
    ob = O.OracleBatch("extended", n, 2)
    assert np.array_equal(h.numpy(), ob.state.encode_symbolic())
    with pytest.raises(ValueError, match="not attached"):
        _lib.check(_lib.lib().gr_host_obs_detach(gb.h, ctypes.c_void_p(12345)))
    _lib.check(_lib.lib().gr_host_obs_detach(gb.h, p))


def test_potion_ties_match_reference(torch_cuda):
    """worldgen.py:647-649 on the device: worlds whose six potion draws tie get
    numpy's (unstable) argsort order, as the reference produced it
    (tests/golden/numpy_corners.npz)."""
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200.levels import LevelBuffer
    g = np.load(os.path.join(GOLD, "numpy_corners.npz"))
    seeds = g["tie_seeds"]
    gb = GridrogueBatch(4, "extended", 0, "symbolic")
    gb.reset()
    lv = LevelBuffer(gb, len(seeds))
    lv.set_params(0, seeds)
    lv.generate(0, len(seeds))
    for k, s in enumerate(seeds):
        assert np.array_equal(lv.world(k)["potion"], g["tie_potion"][k]), f"seed {s}"
    assert gb.worldgen_counters()["potion_ties"] >= len(seeds)


def test_device_argsort6_all_tie_patterns(torch_cuda):
    """np.argsort of six float32 in numpy's tie order, on the device, over all
    6^6 value patterns (tests/golden/numpy_corners.npz)."""
    import itertools
    from paper_2402_16801_b200._lib import check, lib
    from tests._digest import digest
    torch = torch_cuda
    g = np.load(os.path.join(GOLD, "numpy_corners.npz"))
    pats = torch.tensor(list(itertools.product(range(6), repeat=6)), dtype=torch.float32, device="cuda")
    out = torch.empty(pats.shape, dtype=torch.uint8, device="cuda")
    check(lib().gr_selftest_argsort6(pats.data_ptr(), out.data_ptr(), pats.shape[0], None))
    o = out.cpu().numpy().astype(np.int64)
    assert np.array_equal(o[::97], g["argsort6_sample"])
    assert digest(o) == int(g["argsort6_digest"])


def test_device_glibc_sincos_equals_numpy(torch_cuda):
    """Hazard H3: the device's float64 sin / cos (the cave gradients) equal
    numpy's -- glibc's -- bit for bit: on the golden's hard cases (angles where
    glibc is not correctly rounded, minted here) and on EVERY float32 angle in
    [0, 2*pi] against numpy evaluated on this box's host."""
    from paper_2402_16801_b200._lib import check, lib
    from tests._digest import digest
    torch = torch_cuda
    g = np.load(os.path.join(GOLD, "numpy_corners.npz"))

    def dev(x_np):
        x = torch.from_numpy(x_np).cuda()
        s = torch.empty(x.shape, dtype=torch.float64, device="cuda")
        c = torch.empty_like(s)
        check(lib().gr_selftest_sincos64(x.data_ptr(), s.data_ptr(), c.data_ptr(), x.numel(), None))
        return s.cpu().numpy(), c.cpu().numpy()

    s, c = dev(g["trig_x"])
    assert digest(s) == int(g["trig_digest"][0]) and digest(c) == int(g["trig_digest"][1])
    lo, hi = int(np.float32(0).view(np.uint32)), int(np.float32(2 * np.pi).view(np.uint32))
    bad = 0
    for a in range(lo, hi + 1, 1 << 26):
        x = np.arange(a, min(a + (1 << 26), hi + 1), dtype=np.uint32).view(np.float32)
        s, c = dev(x)
        xd = x.astype(np.float64)
        bad += int((s.view(np.uint64) != np.sin(xd).view(np.uint64)).sum())
        bad += int((c.view(np.uint64) != np.cos(xd).view(np.uint64)).sum())
    assert bad == 0


def test_template_floors_match_reference(torch_cuda):
    """worldgen.py:549-595 on the device: with MAX_GEN_RETRIES = 0
    (gr_set_worldgen_attempts) every floor is the template; chests / potions
    over them equal the reference's (tests/golden/template_worlds.npz)."""
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200._lib import check, lib
    from paper_2402_16801_b200.levels import LevelBuffer
    g = np.load(os.path.join(GOLD, "template_worlds.npz"))
    for tier, seeds in (("classic", [0, 7]), ("extended", [0, 7, 123])):
        gb = GridrogueBatch(4, tier, 0, "symbolic")
        gb.reset()
        check(lib().gr_set_worldgen_attempts(gb.h, 0))
        lv = LevelBuffer(gb, len(seeds))
        lv.set_params(0, seeds)
        lv.generate(0, len(seeds))
        for k, s in enumerate(seeds):
            w, tag = lv.world(k), f"{tier}_{s}"
            for key in ("blocks", "items", "spawn", "ladders", "chests", "potion"):
                assert np.array_equal(w[key], g[f"{tag}_{key}"]), f"{tag} {key}"
        assert gb.worldgen_counters()["template_floors"] == len(seeds) * (1 if tier == "classic" else 9)


def _graph_worker(port, q):
    import torch
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        from paper_2402_16801_b200 import GridrogueBatch, ShardedBatch
        n, seed = 2048, 23
        sb = ShardedBatch(n, "extended", seed, "symbolic", max_episode_length=20, graph=True)
        ref = GridrogueBatch(n, "extended", seed, "symbolic", 20, newly=False, info=False)
        sb.reset()
        ref.reset()
        ref.set_validate(False)
        l0 = sb.batch.kernel_launches()
        for k in range(30):
            sb.batch.random_actions(seed, k)
            obs, rew, done, *_ = sb.step(sb.batch.actions)
            ref.random_actions(seed, k)
            o2, r2, d2, *_ = ref.step(ref.actions)
            assert torch.equal(obs, o2) and torch.equal(rew, r2) and torch.equal(done, d2), f"step {k}"
        assert sb._graph is not None, "the sharded step was not captured"
        assert sb.batch.step_index == ref.step_index == 30
        assert sb.batch.kernel_launches() - l0 >= 30 * 5
        st = sb.stats()
        assert st["episodes"] == ref.stats()["episodes"] > 0
        q.put("ok")
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put(traceback.format_exc())


def test_sharded_step_graph_with_nccl(torch_cuda):
    """gr_step_local + the NCCL all-gather + gr_step_finish captured in ONE
    CUDA graph (ShardedBatch(graph=True), world size 1 on this GPU) replays
    the same steps as the plain one-shard path, and the host-side step index
    and launch count stay exact (gr_account_replay)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_graph_worker, args=(29400 + os.getpid() % 200, q))
    p.start()
    msg = q.get(timeout=600)
    p.join(timeout=60)
    assert msg == "ok", msg


def _gold_blob(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("tag,seed,attempts", [("classic_3", 3, 16), ("extended_77", 77, 16),
                                               ("extended_template_7", 7, 0)])
def test_device_world_written_as_reference_bytes(torch_cuda, tag, seed, attempts):
    """serialize.world_to_bytes of a world the device generated is the blob the
    reference's world_to_bytes wrote (serialize.py:77-94), byte for byte."""
    from paper_2402_16801_b200 import GridrogueBatch, serialize as S
    from paper_2402_16801_b200._lib import check, lib
    from paper_2402_16801_b200.levels import LevelBuffer
    tier = tag.split("_")[0]
    gb = GridrogueBatch(2, tier, 0, "symbolic")
    gb.reset()
    check(lib().gr_set_worldgen_attempts(gb.h, attempts))
    lv = LevelBuffer(gb, 1)
    lv.set_params(0, [seed])
    lv.generate(0, 1)
    w = lv.export_world(0)
    assert S.world_to_bytes(w) == _gold_blob(f"world_{tag}.bin")
    if seed == 77:
        assert S.params_to_bytes(lv.level_params(0)) == _gold_blob("level_params_77.bin")


@pytest.mark.parametrize("tag", ["classic_3", "extended_77", "extended_rswap_5", "extended_template_7"])
def test_reference_world_blob_installs_like_reference(torch_cuda, tag):
    """world_from_bytes of a reference blob -> LevelBuffer.import_world ->
    install into an env slot gives the SimState the reference's engine.reset
    gives for that world and key (state.py:169-249); export_world writes the
    blob back byte for byte."""
    from paper_2402_16801_b200 import GridrogueBatch, serialize as S
    from paper_2402_16801_b200.layout import field_shapes, FIELD_NAMES
    from paper_2402_16801_b200.levels import LevelBuffer
    tier = tag.split("_")[0]
    blob = _gold_blob(f"world_{tag}.bin")
    ref = np.load(os.path.join(GOLD, f"world_{tag}_installed.npz"))
    gb = GridrogueBatch(3, tier, 0, "symbolic")
    gb.reset()
    lv = LevelBuffer(gb, 2)
    lv.import_world(1, S.world_from_bytes(blob))
    assert S.world_to_bytes(lv.export_world(1)) == blob
    lv.install([2], [1], [int(ref["key"])])
    ex = gb.export_state(field_shapes(tier, 3))
    bad = [f for f in FIELD_NAMES if not np.array_equal(ex[f][2:3], ref[f])]
    assert not bad, f"installed fields differ from the reference: {bad}"


@pytest.mark.parametrize("tier,obs_mode,n,spec,pdl", [
    ("extended", "symbolic", 8192, "0", "1"), ("extended", "pixels", 2048, "0", "1"),
    ("classic", "symbolic", 4096, "1", "1"), ("extended", "symbolic", 1024, "1", "1"),
    ("extended", "pixels", 2048, "1", "1"), ("classic", "pixels", 1024, "1", "1"),
    ("extended", "symbolic", 2048, "1", "0"), ("extended", "none", 2048, "1", "0")])
def test_two_stream_step_equals_serialised_step(torch_cuda, monkeypatch, tier, obs_mode, n, spec, pdl):
    """Race evidence for the two-stream step (compute-sanitizer is not available
    on this GPU pool): the step whose reset chain (compaction, worldgen,
    install, reset-env obs) runs on a side stream beside the main observation
    writer -- replayed as a CUDA graph, with the speculative pool where noted --
    produces the same observations, rewards, dones and full state, step for
    step, as the same batch with everything serialised on one stream, kernel
    by kernel (GR_OVERLAP=0, GR_GRAPH=0, GR_SPEC=0).  Reset stress: every
    episode ends within 10 steps, so every step runs the reset chain.  The
    speculative pass runs either behind k_step as its programmatic dependent
    with the obs writer forked off (pdl 1) or as its own graph root (pdl 0)."""
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200.layout import field_shapes, FIELD_NAMES
    torch = torch_cuda
    monkeypatch.setenv("GR_SPEC", spec)
    monkeypatch.setenv("GR_SPEC_PDL", pdl)
    fast = GridrogueBatch(n, tier, 9, obs_mode, 10)
    for k, v in (("GR_OVERLAP", "0"), ("GR_GRAPH", "0"), ("GR_SPEC", "0"), ("GR_SPEC_PDL", "0")):
        monkeypatch.setenv(k, v)
    slow = GridrogueBatch(n, tier, 9, obs_mode, 10)
    for b in (fast, slow):
        b.reset()
        b.set_validate(False)
    for k in range(120):
        outs = []
        for b in (fast, slow):
            b.random_actions(9, k)
            outs.append([x.clone() for x in b.step(b.actions)[:4]])
        for x, y in zip(*outs):
            assert torch.equal(x, y), f"step {k}"
        if k % 40 == 39:
            sa, sb = fast.export_state(field_shapes(tier, n)), slow.export_state(field_shapes(tier, n))
            bad = [f for f in FIELD_NAMES if not np.array_equal(sa[f], sb[f])]
            assert not bad, f"state differs at step {k}: {bad}"
    assert fast.episodes_completed() == slow.episodes_completed() >= n * 10


@pytest.mark.parametrize("tier", ["classic", "extended"])
@pytest.mark.parametrize("px", [7, 10, 16])
def test_pixels_every_tile_size_match_reference(torch_cuda, tier, px):
    """The device pixel writer at every supported tile size, both tiers,
    against frames rendered by the reference itself (tests/golden/pixels_px.npz)."""
    from paper_2402_16801_b200 import GridrogueBatch
    from tests._digest import digest
    g = np.load(os.path.join(GOLD, "pixels_px.npz"))
    n, steps, seed, ml = (int(g[k]) for k in ("n", "steps", "seed", "max_len"))
    want = g[f"{tier}_{px}"]
    gb = GridrogueBatch(n, tier, seed, "pixels", ml, tile_px=px)
    assert digest(gb.reset().cpu().numpy()) == int(want[0]), "reset"
    for k in range(steps):
        obs = gb.step(gb.random_actions(seed, k))[0]
        assert digest(obs.cpu().numpy()) == int(want[k + 1]), f"step {k}"


@pytest.mark.parametrize("tier", ["extended", "classic"])
def test_host_step_compact_equals_device_obs(torch_cuda, monkeypatch, tier):
    """gr_step_host into a plain (pageable) numpy array with the compact
    transfer (per-row non-zero bitmap + values, expanded on the host) gives
    exactly the device observation, every step, under reset stress -- and so
    does the plain 2 GB copy (GR_HOST_COMPACT=0); words the host array held
    before are all overwritten."""
    import ctypes
    from paper_2402_16801_b200 import GridrogueBatch
    from paper_2402_16801_b200._lib import check, lib
    torch = torch_cuda
    n, seed = 1536, 3
    monkeypatch.setenv("GR_HOST_COMPACT_MIN_MB", "0")   # the compact path at any size
    for compact in ("1", "0"):
        monkeypatch.setenv("GR_HOST_COMPACT", compact)
        host = GridrogueBatch(n, tier, seed, "symbolic", 10)
        dev = GridrogueBatch(n, tier, seed, "symbolic", 10)
        W = host.obs.shape[1]
        obs = np.full((n, W), -7.5, np.float32)            # garbage the transfer must overwrite
        P = lambda a: ctypes.c_void_p(a.ctypes.data)
        rew = np.zeros(n, np.float32); done = np.zeros(n, np.uint8)
        newly = np.zeros((n, host.n_achievements), np.uint8)
        tm = np.zeros(n, np.uint32); fl = np.zeros(n, np.uint8)
        check(lib().gr_reset_host(host.h, P(obs)))
        assert np.array_equal(obs.view(np.uint32), dev.reset().cpu().numpy().view(np.uint32))
        for k in range(40):
            a = dev.random_actions(seed, k).cpu().numpy()
            check(lib().gr_step_host(host.h, P(a), P(obs), P(rew), P(done), P(newly), P(tm), P(fl)))
            o2, r2, d2, *_ = dev.step(torch.from_numpy(a).cuda())
            assert np.array_equal(obs.view(np.uint32), o2.cpu().numpy().view(np.uint32)), f"obs step {k}"
            assert np.array_equal(rew, r2.cpu().numpy()) and np.array_equal(done, d2.cpu().numpy())


def test_obs_to_host_equals_device_obs(torch_cuda, monkeypatch):
    """GridrogueBatch.obs_to_host (gr_obs_to_host: the compact transfer of any
    device observation buffer, used by the sharded e2e path) writes exactly the
    device observation into a numpy array."""
    from paper_2402_16801_b200 import GridrogueBatch
    monkeypatch.setenv("GR_HOST_COMPACT_MIN_MB", "0")
    gb = GridrogueBatch(1000, "extended", 4, "symbolic", 8)
    gb.reset()
    host = np.full(tuple(gb.obs.shape), 3.25, np.float32)
    for k in range(20):
        obs = gb.step(gb.random_actions(4, k))[0]
        gb.obs_to_host(host)
        assert np.array_equal(host.view(np.uint32), obs.cpu().numpy().view(np.uint32)), f"step {k}"


@pytest.mark.parametrize("tier,px", [("extended", 10), ("classic", 7), ("extended", 16)])
def test_host_pixels_row_classes_equal_device_frames(torch_cuda, monkeypatch, tier, px):
    """Pixel frames into a plain numpy array through the class-row transfer
    (one row per row class gathered on the device, replicated by host threads)
    equal the device frames byte for byte, every step, under reset stress."""
    from paper_2402_16801_b200 import GridrogueBatch
    torch = torch_cuda
    monkeypatch.setenv("GR_HOST_COMPACT_MIN_MB", "0")
    n, seed = 600, 6
    host = GridrogueBatch(n, tier, seed, "pixels", 10, tile_px=px)
    dev = GridrogueBatch(n, tier, seed, "pixels", 10, tile_px=px)
    out = np.full(tuple(host.obs.shape), 77, np.uint8)
    host.reset()
    assert np.array_equal(host.obs_to_host(out), dev.reset().cpu().numpy())
    for k in range(25):
        host.step(host.random_actions(seed, k))
        o2 = dev.step(dev.random_actions(seed, k))[0]
        assert np.array_equal(host.obs_to_host(out), o2.cpu().numpy()), f"step {k}"


@pytest.mark.parametrize("tier,obs_mode,px,n,offset", [
    ("extended", "symbolic", None, 700, 0), ("extended", "symbolic", None, 700, 4),
    ("classic", "symbolic", None, 523, 12), ("extended", "pixels", 10, 301, 0),
    ("extended", "pixels", 10, 301, 3), ("classic", "pixels", 7, 259, 1),
    ("extended", "pixels", 16, 77, 9), ("extended", "pixels", 7, 101, 14)])
def test_writers_stay_inside_the_observation_buffer(torch_cuda, tier, obs_mode, px, n, offset):
    """Out-of-bounds evidence without compute-sanitizer (closed on this GPU
    pool): the observation buffer is a view into a larger allocation whose
    guard bands hold a fill pattern, at 16-byte-aligned and unaligned starts
    (the writers take TMA / 16-byte stores from the aligned address at or
    below the buffer); every step under reset stress, the guard bands stay
    untouched and the frames equal a normally allocated twin's."""
    from paper_2402_16801_b200 import GridrogueBatch
    torch = torch_cuda
    kw = {"tile_px": px} if px else {}
    gb = GridrogueBatch(n, tier, 5, obs_mode, 9, **kw)
    twin = GridrogueBatch(n, tier, 5, obs_mode, 9, **kw)
    nbytes = gb.obs.numel() * gb.obs.element_size()
    G = 4096
    big = torch.full((nbytes + 2 * G,), 0xA5, dtype=torch.uint8, device="cuda")
    gb.obs = big[G + offset:G + offset + nbytes].view(gb.obs.dtype).view(gb.obs.shape)
    guard = lambda: (big[:G + offset].eq(0xA5).all().item() and big[G + offset + nbytes:].eq(0xA5).all().item())
    gb.reset()
    assert torch.equal(gb.obs, twin.reset()) and guard()
    for k in range(30):
        gb.step(gb.random_actions(5, k))
        twin.step(twin.random_actions(5, k))
        assert guard(), f"guard band written at step {k}"
        assert torch.equal(gb.obs.view(torch.uint8), twin.obs.view(torch.uint8)), f"step {k}"
