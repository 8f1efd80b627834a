"""Multi-GPU sharding: one process per GPU, each owning a contiguous slice
of the global batch.

Every env is independent, but the reference's batch couples envs in three
places: the optimistic-reset pool slot is the *global* rank of each done
env mod M (batch.py:224), and two `any()` flags span the whole batch
(creatures.py:290,329 cooldown decrement; obs.py:236 torch glow).  One
int32[4] record per rank -- [done count, flags, 0, 0] -- is all-gathered per
step (NCCL over NVLink; gloo in the CPU tests) and combined exactly like
``combine_exchange`` below (device twin: k_finish_info in gr_reset.cu).
Episode statistics are all-reduced only when read (K9 of SURVEY.md).
"""

from __future__ import annotations

import numpy as np


def shard_bounds(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of env indices owned by ``rank``."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, rem = divmod(n_global, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def combine_exchange(records: np.ndarray, rank: int, pool_size: int) -> dict:
    """Host twin of k_finish_info: records is int32[world, 4]."""
    rec = np.asarray(records, np.int64).reshape(-1, 4)
    k = int(rec[rank, 0])
    return {"k_local": k, "offset": int(rec[:rank, 0].sum()),
            "n_pool": min(k, pool_size), "flags": int(np.bitwise_or.reduce(rec[:, 1]))}


class ShardedBatch:
    """This rank's shard of a globally-consistent batch."""

    def __init__(self, n_envs_global: int, tier: str = "extended", seed: int = 0,
                 obs_mode: str = "symbolic", max_episode_length: int | None = None,
                 tile_px: int | None = None, reset_ratio: int = 16, group=None, device=None,
                 graph: bool = False):
        import os
        import torch
        import torch.distributed as dist
        from .env import GridrogueBatch
        # ranks of one node share its host cores: the host threads of the
        # compact / delta observation transfers get an equal share each
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        if local_world > 1:
            os.environ.setdefault("GR_HOST_THREADS", str(max(1, (os.cpu_count() or 1) // local_world)))
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.lo, self.hi = shard_bounds(n_envs_global, self.world, self.rank)
        dev = torch.cuda.current_device() if device is None else device
        self.batch = GridrogueBatch(self.hi - self.lo, tier, seed, obs_mode, max_episode_length,
                                    tile_px, dev, reset_ratio, env_offset=self.lo,
                                    n_envs_global=n_envs_global)
        self.ex = torch.zeros(4, dtype=torch.int32, device=self.batch.device)
        self.ex_all = torch.zeros(4 * self.world, dtype=torch.int32, device=self.batch.device)
        # graph=True (NCCL): after two eager steps, gr_step_local + the NCCL
        # all-gather + gr_step_finish are captured in ONE CUDA graph and
        # replayed (action validation off: the device policy's actions are
        # valid by construction; validation would synchronise the stream)
        self.graph = bool(graph)
        self._graph = None
        self._eager_steps = 0
        self._launches_per_step = 0
        if self.graph:
            self.batch.set_validate(False)

    def reset(self):
        return self.batch.reset()

    def random_actions(self, seed: int, t: int):
        return self.batch.random_actions(seed, t)

    def step(self, actions=None):
        a = self.batch.actions if actions is None else actions
        if a is not self.batch.actions:
            self.batch.actions.copy_(a)   # int64, on this rank's device
            a = self.batch.actions
        if self._graph is not None:
            from ._lib import check, lib
            self._graph.replay()
            check(lib().gr_account_replay(self.batch.h, 1, self._launches_per_step))
            return self._outputs()
        if self.graph and self._eager_steps >= 2:
            return self._capture_and_run(a)
        self._eager_steps += 1
        return self._step_eager(a)

    def _step_eager(self, a):
        self.batch.step_local(a, self.ex)
        self.dist.all_gather_into_tensor(self.ex_all, self.ex, group=self.group)
        return self.batch.step_finish(self.ex_all, self.rank, self.world)

    def _outputs(self):
        b = self.batch
        return b.obs, b.reward, b.done, b.newly, b.time, b.floor

    def _collective_capturable(self) -> bool:
        """Whether this process group's all-gather can be captured in a CUDA
        graph here (probed on scratch tensors, so a failure touches no state)."""
        import torch
        try:
            src = torch.zeros(4, dtype=torch.int32, device=self.batch.device)
            dst = torch.zeros(4 * self.world, dtype=torch.int32, device=self.batch.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.dist.all_gather_into_tensor(dst, src, group=self.group)
            g.replay()
            torch.cuda.synchronize(self.batch.device)
            return True
        except Exception as ex:   # keep stepping eagerly rather than fail the run
            import warnings
            warnings.warn(f"ShardedBatch: collective not capturable here ({ex}); stepping without a graph")
            return False

    def _capture_and_run(self, a):
        """Capture local step + all-gather + finish once, then replay.  The
        library's host-side bookkeeping advanced once during the capture; that
        advance stands for the first replay, issued right after."""
        import torch
        if not self._collective_capturable():
            self.graph = False
            return self._step_eager(a)
        l0 = self.batch.kernel_launches()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step_eager(a)
        self._launches_per_step = self.batch.kernel_launches() - l0
        self._graph = g
        g.replay()
        return self._outputs()

    def stats(self) -> dict:
        import torch
        s = self.batch.stats()
        v = torch.tensor([s["episodes"], s["total_steps"], *s["ach_episodes"]], dtype=torch.float64,
                         device=self.batch.device)
        r = torch.tensor([s["total_return"]], dtype=torch.float64, device=self.batch.device)
        self.dist.all_reduce(v, group=self.group)
        self.dist.all_reduce(r, group=self.group)
        v = v.cpu().numpy()
        return {"episodes": int(v[0]), "total_steps": int(v[1]), "total_return": float(r.item()),
                "ach_episodes": v[2:].astype(np.int64)}
