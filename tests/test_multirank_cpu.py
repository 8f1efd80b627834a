"""The N>1 path on CPU: two gloo ranks, each owning a contiguous shard.

Every rank runs the oracle restricted to its shard (global env indices for
worldgen and the policy, global pool size) and the batch-coupled quantities
travel through torch.distributed exactly as in ShardedBatch: the per-rank
exchange record is all-gathered and combined by
``paper_2402_16801_b200.parallel.combine_exchange`` (the host twin of the
device kernel k_finish_info).  The concatenated shards must equal one
global batch bit for bit -- rewards, dones, symbolic obs, every state field
and the episode statistics.
"""

import os
import socket

import numpy as np
import pytest

from tests._digest import digest


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, tier, n_global, steps, seed, max_len, out_dir):
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_2402_16801_b200.parallel import shard_bounds, combine_exchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(n_global, world, rank)
    n = hi - lo
    b = O.OracleBatch(tier, n, seed, max_episode_length=max_len, env_offset=lo, n_global=n_global)
    M = max(1, -(-n_global // 16))
    na = O.TIERS[tier]["NA"]
    rec = {"reward": [], "done": [], "obs": [], "k": []}
    for t in range(steps):
        a = O.random_actions(seed, t, n, na, env0=lo)
        fl = torch.from_numpy(b.step_a(a).astype(np.int32))
        allfl = [torch.zeros(2, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allfl, fl)
        gfl = np.bitwise_or.reduce(np.stack([x.numpy() for x in allfl]), axis=0)
        r, d, nw, info, k = b.step_b(gfl)
        record = torch.tensor([k, 0, 0, 0], dtype=torch.int32)
        allrec = [torch.zeros(4, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allrec, record)
        ex = combine_exchange(np.stack([x.numpy() for x in allrec]), rank, M)
        assert ex["k_local"] == k
        b.step_c(ex["offset"])
        dk = torch.tensor([int(b.any_dark())], dtype=torch.int32)
        dist.all_reduce(dk, op=dist.ReduceOp.MAX)
        rec["reward"].append(r)
        rec["done"].append(d)
        rec["obs"].append(b.encode_symbolic(bool(dk.item())))
        rec["k"].append(k)
    state = b.state.export_fields()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=lo, hi=hi,
             reward=np.stack(rec["reward"]), done=np.stack(rec["done"]),
             obs_digest=np.array([digest(o) for o in rec["obs"]], np.uint64),
             obs_last=rec["obs"][-1], episodes=b.stats()["episodes"],
             **{f"f_{k}": v for k, v in state.items()})
    dist.destroy_process_group()


@pytest.mark.parametrize("tier,n_global,steps,max_len", [
    ("classic", 51, 90, 40),
    ("extended", 34, 60, 25),
])
def test_two_rank_shards_equal_global_batch(tmp_path, oracle_lib, tier, n_global, steps, max_len):
    import torch.multiprocessing as mp
    O = oracle_lib
    world, seed = 2, 3
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, tier, n_global, steps, seed, max_len, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    g = O.OracleBatch(tier, n_global, seed, max_episode_length=max_len)
    na = O.TIERS[tier]["NA"]
    total_eps = sum(int(p["episodes"]) for p in parts)
    for t in range(steps):
        r, d, _, _ = g.step(O.random_actions(seed, t, n_global, na))
        assert np.array_equal(r, np.concatenate([p["reward"][t] for p in parts])), f"reward step {t}"
        assert np.array_equal(d, np.concatenate([p["done"][t] for p in parts])), f"done step {t}"
    obs = g.state.encode_symbolic()
    assert np.array_equal(obs, np.concatenate([p["obs_last"] for p in parts]))
    gs = g.state.export_fields()
    for f in O.FIELD_NAMES:
        assert np.array_equal(gs[f], np.concatenate([p[f"f_{f}"] for p in parts])), f
    assert g.stats()["episodes"] == total_eps
    assert total_eps > n_global // 2     # the pool path was exercised across shards
