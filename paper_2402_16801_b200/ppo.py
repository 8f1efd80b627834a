"""PPO on the device batch engine: the caller of the hot path.

Craftax-1B's PPO (PAPER.md, "Hyperparameter Tuning", Craftax-1B table):
1024 env workers, 64 steps per rollout, 8 minibatches, 4 update epochs,
MLP layer size 512 with tanh, learning rate 2e-4 linearly annealed, gamma
0.99, GAE lambda 0.8, clip 0.2, value coefficient 0.5, entropy coefficient
0.01.  Actor and critic are separate 3-hidden-layer MLPs (orthogonal init,
gain sqrt 2; 0.01 on the policy head, 1 on the value head), Adam (eps 1e-5),
global gradient-norm clip 0.5 -- the purejaxrl recipe the paper builds on.
The reference ships no learner, so there is nothing to match
bit for bit; tests check the advantage estimator against a plain loop and
that a short run learns (tests/test_ppo_cpu.py, tests/test_gpu.py).

Everything stays on the GPU: the CUDA writer renders observations into the
batch's device buffer, copied on the device into the rollout buffer (one
stable set of buffer addresses keeps every env step a replay of the
library's captured step graph); actions go back as a device tensor.  Multi-GPU: one process per GPU (torchrun), each with its own
shard of the global batch (parallel.ShardedBatch, so pools and resets match
one global batch), gradients all-reduced over NCCL by DDP.

    python -m paper_2402_16801_b200.ppo --total-timesteps 20000000
    python -m paper_2402_16801_b200.ppo --gpus 8 --total-timesteps 1000000000
    (--gpus N re-launches itself under torch.distributed.run, one rank per GPU;
    torchrun --nproc-per-node 8 -m paper_2402_16801_b200.ppo ... is equivalent)
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from dataclasses import asdict, dataclass

import numpy as np


@dataclass
class PPOConfig:
    tier: str = "extended"
    n_envs: int = 1024            # per GPU
    n_steps: int = 64
    n_minibatches: int = 8
    update_epochs: int = 4
    layer_size: int = 512
    lr: float = 2e-4
    anneal_lr: bool = True
    gamma: float = 0.99
    gae_lambda: float = 0.8
    clip_eps: float = 0.2
    vf_coef: float = 0.5
    ent_coef: float = 0.01
    max_grad_norm: float = 0.5
    total_timesteps: int = 1_000_000_000
    seed: int = 0
    bf16: bool = True             # autocast the MLPs to bf16 (tensor cores)
    graphs: bool = True           # one GPU: rollout step, GAE and minibatch update as CUDA graphs
    fused_loss: bool = True       # graphed learner: PPO objective + gradient in one CUDA kernel (gr_ppo.cu)
    fused_sampler: bool = True    # graphed learner: action sampling + rollout-buffer writes in one kernel
    manual_backward: bool = True  # graphed bf16 learner: hand-written backward + clip/Adam kernels (learner.py)


def gae(rewards, values, dones, last_value, gamma: float, lam: float):
    """Generalized advantage estimation over a [T, N] rollout.

    dones[t] marks that the episode ended at step t (the env auto-reset), so
    value[t + 1] belongs to a new episode and is not bootstrapped.
    """
    import torch
    T = rewards.shape[0]
    adv = torch.zeros_like(rewards)
    last = torch.zeros_like(last_value)
    for t in range(T - 1, -1, -1):
        nxt = last_value if t == T - 1 else values[t + 1]
        nonterm = 1.0 - dones[t]
        delta = rewards[t] + gamma * nxt * nonterm - values[t]
        last = delta + gamma * lam * nonterm * last
        adv[t] = last
    return adv, adv + values


def _mlp(nn, sizes, out, out_gain):
    layers = []
    for a, b in zip(sizes[:-1], sizes[1:]):
        lin = nn.Linear(a, b)
        nn.init.orthogonal_(lin.weight, math.sqrt(2))
        nn.init.zeros_(lin.bias)
        layers += [lin, nn.Tanh()]
    head = nn.Linear(sizes[-1], out)
    nn.init.orthogonal_(head.weight, out_gain)
    nn.init.zeros_(head.bias)
    return nn.Sequential(*layers, head)


def make_model(obs_dim: int, n_actions: int, layer: int):
    import torch.nn as nn

    class ActorCritic(nn.Module):
        def __init__(self):
            super().__init__()
            self.actor = _mlp(nn, [obs_dim, layer, layer, layer], n_actions, 0.01)
            self.critic = _mlp(nn, [obs_dim, layer, layer, layer], 1, 1.0)

        def forward(self, x):
            return self.actor(x), self.critic(x).squeeze(-1)

    return ActorCritic()


def make_fused_model(obs_dim: int, n_actions: int, layer: int):
    """The same actor and critic as make_model, with the two first layers
    stored as one [2*layer, obs_dim] weight (rows [0, layer) the actor's, the
    rest the critic's, each half orthogonally initialised on its own): one
    GEMM over the wide observation instead of two.  Mathematically the two
    separate MLPs."""
    import torch
    import torch.nn as nn

    class FusedActorCritic(nn.Module):
        def __init__(self):
            super().__init__()
            self.layer = layer
            self.first = nn.Linear(obs_dim, 2 * layer)
            with torch.no_grad():
                for h in range(2):
                    nn.init.orthogonal_(self.first.weight[h * layer:(h + 1) * layer], math.sqrt(2))
                nn.init.zeros_(self.first.bias)
            self.actor = _mlp(nn, [layer, layer, layer], n_actions, 0.01)
            self.critic = _mlp(nn, [layer, layer, layer], 1, 1.0)

        def forward(self, x):
            h = torch.tanh(self.first(x))
            return self.actor(h[:, :self.layer]), self.critic(h[:, self.layer:]).squeeze(-1)

    return FusedActorCritic()


def train(cfg: PPOConfig, log=print, max_updates: int | None = None) -> dict:
    import torch
    import torch.distributed as dist
    from .env import TIERS, GridrogueBatch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    if cfg.graphs:
        return _train_graphed(cfg, log, max_updates)
    torch.manual_seed(cfg.seed + rank)

    n, T = cfg.n_envs, cfg.n_steps
    if world > 1:
        from .parallel import ShardedBatch
        env = ShardedBatch(n * world, cfg.tier, cfg.seed, "symbolic")
        gb = env.batch
    else:
        env = gb = GridrogueBatch(n, cfg.tier, cfg.seed, "symbolic", newly=False, info=False)
    gb.set_validate(False)   # actions are sampled in range
    t_info = TIERS[cfg.tier]
    obs_dim, n_actions = t_info["obs"], t_info["n_actions"]

    model = make_model(obs_dim, n_actions, cfg.layer_size).to(dev)
    if world > 1:
        model = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local])
    opt = torch.optim.Adam(model.parameters(), lr=cfg.lr, eps=1e-5)
    batch_size = n * T
    n_updates = max(1, cfg.total_timesteps // (batch_size * world))
    if max_updates is not None:
        n_updates = min(n_updates, max_updates)
    mb = batch_size // cfg.n_minibatches

    buf_obs = torch.empty((T, n, obs_dim), dtype=torch.float32, device=dev)
    buf_act = torch.empty((T, n), dtype=torch.int64, device=dev)
    buf_logp = torch.empty((T, n), dtype=torch.float32, device=dev)
    buf_val = torch.empty((T, n), dtype=torch.float32, device=dev)
    buf_rew = torch.empty((T, n), dtype=torch.float32, device=dev)
    buf_done = torch.empty((T, n), dtype=torch.float32, device=dev)

    def policy(x):
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=cfg.bf16):
            logits, v = model(x)
        return logits.float(), v.float()

    obs = env.reset().clone()
    history = []
    last_ep, last_ret = 0, 0.0
    t0 = time.perf_counter()
    steps_done = 0
    for upd in range(n_updates):
        if cfg.anneal_lr:
            for g in opt.param_groups:
                g["lr"] = cfg.lr * (1.0 - upd / n_updates)
        # --- rollout ---------------------------------------------------------
        with torch.no_grad():
            for t in range(T):
                buf_obs[t].copy_(obs)
                logits, v = policy(obs)
                dist_ = torch.distributions.Categorical(logits=logits)
                a = dist_.sample()
                buf_act[t] = a
                buf_logp[t] = dist_.log_prob(a)
                buf_val[t] = v
                out = env.step(a)
                obs, rew, done = out[0], out[1], out[2]
                buf_rew[t] = rew
                buf_done[t] = done.float()
            _, last_v = policy(obs)
            adv, ret = gae(buf_rew, buf_val, buf_done, last_v, cfg.gamma, cfg.gae_lambda)
        obs = obs.clone()   # the env overwrites its obs tensor in place next step
        # --- update ----------------------------------------------------------
        b_obs = buf_obs.reshape(batch_size, obs_dim)
        b_act, b_logp = buf_act.reshape(-1), buf_logp.reshape(-1)
        b_adv, b_ret, b_val = adv.reshape(-1), ret.reshape(-1), buf_val.reshape(-1)
        stats = []
        for _ in range(cfg.update_epochs):
            perm = torch.randperm(batch_size, device=dev)
            for k in range(cfg.n_minibatches):
                idx = perm[k * mb:(k + 1) * mb]
                logits, v = policy(b_obs[idx])
                d = torch.distributions.Categorical(logits=logits)
                logp = d.log_prob(b_act[idx])
                ratio = torch.exp(logp - b_logp[idx])
                a_ = b_adv[idx]
                a_ = (a_ - a_.mean()) / (a_.std() + 1e-8)
                pg = -torch.min(ratio * a_, ratio.clamp(1 - cfg.clip_eps, 1 + cfg.clip_eps) * a_).mean()
                v_clip = b_val[idx] + (v - b_val[idx]).clamp(-cfg.clip_eps, cfg.clip_eps)
                vl = 0.5 * torch.max((v - b_ret[idx]) ** 2, (v_clip - b_ret[idx]) ** 2).mean()
                ent = d.entropy().mean()
                loss = pg + cfg.vf_coef * vl - cfg.ent_coef * ent
                opt.zero_grad(set_to_none=True)
                loss.backward()
                torch.nn.utils.clip_grad_norm_(model.parameters(), cfg.max_grad_norm)
                opt.step()
                stats.append(torch.stack([loss.detach(), pg.detach(), vl.detach(), ent.detach()]))
        steps_done += batch_size * world
        if upd % 10 == 0 or upd == n_updates - 1:
            torch.cuda.synchronize()
            s = torch.stack(stats).mean(0).tolist()
            st = gb.stats()
            mean_ret = st["total_return"] / max(st["episodes"], 1)
            window = (st["total_return"] - last_ret) / max(st["episodes"] - last_ep, 1)
            last_ep, last_ret = st["episodes"], st["total_return"]
            row = {"update": upd, "env_steps": steps_done, "sps": round(steps_done / (time.perf_counter() - t0), 1),
                   "loss": s[0], "pg_loss": s[1], "v_loss": s[2], "entropy": s[3],
                   "episodes": st["episodes"], "mean_episode_return": mean_ret,
                   "recent_episode_return": window}
            history.append(row)
            if rank == 0:
                log(json.dumps(row))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = gb.stats()
    result = {"config": asdict(cfg), "n_gpus": world, "updates": n_updates, "env_steps": steps_done,
              "seconds": round(dt, 3), "sps": round(steps_done / dt, 1), "episodes_rank0": st["episodes"],
              "mean_episode_return_rank0": st["total_return"] / max(st["episodes"], 1), "history": history}
    return result


_OBJECTIVE = None


def _objective_fn():
    """torch.autograd.Function over the fused kernel (built once)."""
    global _OBJECTIVE
    if _OBJECTIVE is not None:
        return _OBJECTIVE
    import torch
    from ._lib import lib

    class _Objective(torch.autograd.Function):
        @staticmethod
        def forward(ctx, z, v, actions, logp_old, adv, values_old, returns, clip_eps, vf_coef, ent_coef):
            B, NA = z.shape
            dz = torch.empty_like(z)
            dv = torch.empty_like(v)
            out = torch.zeros(4, dtype=torch.float32, device=z.device)
            stream = torch.cuda.current_stream(z.device).cuda_stream
            rc = lib().grp_ppo_loss(z.data_ptr(), v.data_ptr(), actions.data_ptr(), logp_old.data_ptr(),
                                    adv.data_ptr(), values_old.data_ptr(), returns.data_ptr(), B, NA,
                                    clip_eps, vf_coef, ent_coef, dz.data_ptr(), dv.data_ptr(), out.data_ptr(),
                                    stream)
            if rc != 0:
                raise RuntimeError(f"grp_ppo_loss failed ({rc}): n_actions {NA}, batch {B}")
            ctx.save_for_backward(dz, dv)
            loss = out[0].clone()
            ctx.mark_non_differentiable(out)
            return loss, out

        @staticmethod
        def backward(ctx, g_loss, g_out):
            dz, dv = ctx.saved_tensors
            return dz * g_loss, dv * g_loss, None, None, None, None, None, None, None, None

    _OBJECTIVE = _Objective
    return _OBJECTIVE


def ppo_objective(logits, values, actions, logp_old, adv, values_old, returns, clip_eps: float,
                  vf_coef: float, ent_coef: float):
    """The PPO minibatch objective through the fused kernel
    (include/gridrogue_ppo.h): returns (loss, stats = [loss, pg, vl,
    entropy]); d loss / d logits and d loss / d values come from the same
    launch.  The advantages are normalised over the minibatch inside."""
    z = logits.float().contiguous()
    v = values.float().contiguous()
    args = [t.contiguous() for t in (actions, logp_old, adv, values_old, returns)]
    return _objective_fn().apply(z, v, *args, float(clip_eps), float(vf_coef), float(ent_coef))


def _train_graphed(cfg: PPOConfig, log, max_updates: int | None) -> dict:
    """Single-GPU PPO with every per-step launch sequence replayed as a CUDA graph.

    The eager loop in train() issues ~40 small kernels per env step and
    ~150 per minibatch from Python; at Craftax-1B's 1,024 envs the GPU then
    idles between launches.  Here, after one eager warm-up update:
      * rollout step t = one graph (obs -> bf16 rollout buffer, actor / critic
        forward, Gumbel-max sample into the env's action buffer, log-prob,
        value, the previous step's reward / done), then the env step (the
        library's own captured step graph);
      * GAE over the rollout = one graph;
      * the whole update = one graph: per epoch a device permutation, then
        per minibatch the gather, forward, the fused PPO objective
        (gr_ppo.cu: loss and its logits / value gradients in one kernel),
        backward, global-norm clip and Adam with a device-side learning rate.
    Several GPUs (torchrun, one process each): every rank owns a shard of
    the global batch (parallel.ShardedBatch); each minibatch is then two
    graphs around one all-reduce of a flat gradient buffer (the parameters'
    .grad tensors are views into it), the average taken in the second graph.
    Same algorithm and hyper-parameters as the eager loop; the sampling
    noise comes from counter-based hashes (Gumbel-max), so runs are not
    bitwise equal to eager ones.
    """
    import torch
    from .env import TIERS, GridrogueBatch

    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    torch.manual_seed(cfg.seed)   # the same initial weights on every rank
    n, T = cfg.n_envs, cfg.n_steps
    if world > 1:
        from .parallel import ShardedBatch
        env = ShardedBatch(n * world, cfg.tier, cfg.seed, "symbolic")
        gb = env.batch
    else:
        env = gb = GridrogueBatch(n, cfg.tier, cfg.seed, "symbolic", newly=False, info=False)
    gb.set_validate(False)   # actions are sampled in range
    t_info = TIERS[cfg.tier]
    obs_dim, n_actions = t_info["obs"], t_info["n_actions"]
    # rows padded to a multiple of 64 elements (8268 -> 8320): cuBLAS runs the
    # first layer's GEMMs on its fast tensor-core path only with 16-byte
    # aligned leading dimensions; the pad columns hold zeros, so they add
    # nothing to the pre-activations and their weights get zero gradients
    obs_pad = (obs_dim + 63) // 64 * 64
    batch_size = n * T
    mb = batch_size // cfg.n_minibatches
    manual = cfg.manual_backward and cfg.bf16 and cfg.fused_loss
    learner = None
    if manual:
        from .learner import ManualLearner, pad_actions
        # the action head padded to a multiple of 8 outputs (zero rows that
        # stay zero: their gradients are exactly zero)
        model = make_fused_model(obs_pad, pad_actions(n_actions), cfg.layer_size).to(dev)
        with torch.no_grad():
            model.actor[-1].weight[n_actions:].zero_()
            model.actor[-1].bias[n_actions:].zero_()
        learner = ManualLearner(model, n_actions, mb, dev)
        params = learner.params
        flat_grad = learner.G   # the .grad tensors are views of it
    else:
        model = make_fused_model(obs_pad, n_actions, cfg.layer_size).to(dev)
        params = list(model.parameters())
        # gradients as views of one flat buffer: one all-reduce per minibatch
        flat_grad = torch.zeros(sum(p.numel() for p in params), dtype=torch.float32, device=dev)
        off = 0
        for p_ in params:
            p_.grad = flat_grad[off:off + p_.numel()].view_as(p_)
            off += p_.numel()
    if world > 1:
        for p_ in params:
            dist.broadcast(p_.data, 0)
    if learner is not None:
        learner.Pb.copy_(learner.P)
        # the rollout reads the learner's bf16 weights (refreshed by every Adam step)
        roll_w = learner.bf16_weights()
    else:
        # rollout weights: bf16 copies refreshed once per rollout (the weights do
        # not change within one), so the 64 per-step graphs cast nothing
        roll_w = [p.detach().to(torch.bfloat16 if cfg.bf16 else torch.float32) for p in params]
    lr_t = torch.tensor(cfg.lr, dtype=torch.float32, device=dev)
    opt = None if manual else torch.optim.Adam(params, lr=lr_t, eps=1e-5, capturable=True, fused=True)
    n_updates = max(1, cfg.total_timesteps // (batch_size * world))
    if max_updates is not None:
        n_updates = min(n_updates, max_updates)
    odt = torch.bfloat16 if cfg.bf16 else torch.float32   # autocast casts the input to bf16 anyway

    buf_obs = torch.zeros((T, n, obs_pad), dtype=odt, device=dev)
    last_obs = torch.zeros((n, obs_pad), dtype=odt, device=dev)
    buf_act = torch.empty((T, n), dtype=torch.int64, device=dev)
    buf_logp = torch.empty((T, n), dtype=torch.float32, device=dev)
    buf_val = torch.empty((T, n), dtype=torch.float32, device=dev)
    buf_rew = torch.empty((T, n), dtype=torch.float32, device=dev)
    buf_done = torch.empty((T, n), dtype=torch.float32, device=dev)
    adv = torch.empty((T, n), dtype=torch.float32, device=dev)
    ret = torch.empty((T, n), dtype=torch.float32, device=dev)
    last_v = torch.empty(n, dtype=torch.float32, device=dev)
    idx_s = torch.zeros(mb, dtype=torch.int64, device=dev)
    stats_s = torch.zeros(4, dtype=torch.float32, device=dev)
    stats_acc = torch.zeros(4, dtype=torch.float32, device=dev)

    def policy(x):
        # no autocast weight cache: graphs must own their casts
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=cfg.bf16, cache_enabled=False):
            logits, v = model(x)
        return logits[:, :n_actions].float(), v.float()

    lin_ix = [(k, k + 1) for k in range(0, len(params), 2)]   # (weight, bias) per Linear, module order

    def roll_policy(x):
        ha, hc = roll_policy_raw(x)
        return ha[:, :n_actions].float(), hc.float().squeeze(-1)

    roll_acts = learner.make_acts(n) if learner is not None else None

    def roll_policy_raw(x):
        """Rollout forward on the pre-cast weights (module order: first,
        actor 2 + head, critic 2 + head); logits [N, A] and values [N, 1] in
        the rollout dtype."""
        if learner is not None:   # the learner's forward on its bf16 weights
            return learner.forward(x, roll_acts)
        F = torch.nn.functional
        (w0, b0), rest = lin_ix[0], lin_ix[1:]
        h = torch.tanh(F.linear(x, roll_w[w0], roll_w[b0]))
        L = cfg.layer_size
        ha, hc = h[:, :L], h[:, L:]
        na = (len(rest)) // 2
        for j, (w, b) in enumerate(rest[:na]):
            ha = F.linear(ha, roll_w[w], roll_w[b])
            if j < na - 1:
                ha = torch.tanh(ha)
        for j, (w, b) in enumerate(rest[na:]):
            hc = F.linear(hc, roll_w[w], roll_w[b])
            if j < na - 1:
                hc = torch.tanh(hc)
        return ha, hc

    rng_ctr = torch.zeros(1, dtype=torch.int64, device=dev)   # sampler counter, one per rollout

    def obs_to(dst, obs):
        """A step's float32 observations into a (padded) rollout row block."""
        if dst.dtype == torch.bfloat16:
            from ._lib import lib
            rc = lib().grp_rows_to_bf16(obs.data_ptr(), n, obs_dim, dst.data_ptr(), dst.stride(0),
                                        torch.cuda.current_stream(dev).cuda_stream)
            if rc != 0:
                raise RuntimeError(f"grp_rows_to_bf16 failed ({rc})")
        else:
            dst[:, :obs_dim].copy_(obs)

    def refresh_roll_w():
        if learner is None:
            for dst, src in zip(roll_w, params):
                dst.copy_(src.detach())
        rng_ctr.add_(1)

    def roll_step(t):
        if t > 0 and (t == T or not cfg.fused_sampler):
            buf_rew[t - 1].copy_(gb.reward)
            buf_done[t - 1].copy_(gb.done)
        if t == T:   # closing step: the bootstrap value
            obs_to(last_obs, gb.obs)
            _, v = roll_policy(last_obs)
            last_v.copy_(v)
            return
        obs_to(buf_obs[t], gb.obs)
        if cfg.fused_sampler:
            # sampling, log-prob, value and the previous reward / done in one
            # launch (gr_ppo.cu): the step's other ~15 small kernels
            from ._lib import lib
            za, zv = roll_policy_raw(buf_obs[t])
            prev = t > 0
            rc = lib().grp_sample_actions(
                za.data_ptr(), zv.data_ptr(), 1 if za.dtype == torch.bfloat16 else 0, n, n_actions, za.stride(0),
                zv.stride(0), (cfg.seed * 0x9E3779B97F4A7C15 + 1 + rank * 0xD1B54A32D192ED03) & 0xFFFFFFFFFFFFFFFF, rng_ctr.data_ptr(), t,
                gb.actions.data_ptr(), buf_act[t].data_ptr(), buf_logp[t].data_ptr(), buf_val[t].data_ptr(),
                gb.reward.data_ptr() if prev else None, gb.done.data_ptr() if prev else None,
                buf_rew[t - 1].data_ptr() if prev else None, buf_done[t - 1].data_ptr() if prev else None,
                torch.cuda.current_stream(dev).cuda_stream)
            if rc != 0:
                raise RuntimeError(f"grp_sample_actions failed ({rc})")
            return
        logits, v = roll_policy(buf_obs[t])
        u = torch.rand_like(logits).clamp_(min=1e-20)
        a = (logits - torch.log(-torch.log(u))).argmax(-1)
        logp = torch.log_softmax(logits, -1).gather(-1, a[:, None]).squeeze(-1)
        gb.actions.copy_(a)
        buf_act[t].copy_(a)
        buf_logp[t].copy_(logp)
        buf_val[t].copy_(v)

    def gae_step():
        a_, r_ = gae(buf_rew, buf_val, buf_done, last_v, cfg.gamma, cfg.gae_lambda)
        adv.copy_(a_)
        ret.copy_(r_)

    b_obs = buf_obs.view(batch_size, obs_pad)
    b_act, b_logp = buf_act.view(-1), buf_logp.view(-1)
    b_adv, b_ret, b_val = adv.view(-1), ret.view(-1), buf_val.view(-1)

    x_mb = torch.empty((mb, obs_pad), dtype=odt, device=dev) if learner is not None else None

    def mb_step():
        idx = idx_s
        if learner is not None:
            torch.index_select(b_obs, 0, idx, out=x_mb)
            learner.forward(x_mb)
            learner.loss(b_act, b_logp, b_adv, b_val, b_ret, cfg.clip_eps, cfg.vf_coef, cfg.ent_coef, stats_s,
                         index=idx)
            learner.backward(x_mb)
            return
        logits, v = policy(b_obs.index_select(0, idx))
        if cfg.fused_loss:
            loss, st = ppo_objective(logits, v, b_act.index_select(0, idx), b_logp.index_select(0, idx),
                                     b_adv.index_select(0, idx), b_val.index_select(0, idx),
                                     b_ret.index_select(0, idx), cfg.clip_eps, cfg.vf_coef, cfg.ent_coef)
            loss.backward()
            stats_s.copy_(st)
            return
        logp_all = torch.log_softmax(logits, -1)
        logp = logp_all.gather(-1, b_act.index_select(0, idx)[:, None]).squeeze(-1)
        ratio = torch.exp(logp - b_logp.index_select(0, idx))
        a_ = b_adv.index_select(0, idx)
        a_ = (a_ - a_.mean()) / (a_.std() + 1e-8)
        pg = -torch.min(ratio * a_, ratio.clamp(1 - cfg.clip_eps, 1 + cfg.clip_eps) * a_).mean()
        bv, br = b_val.index_select(0, idx), b_ret.index_select(0, idx)
        v_clip = bv + (v - bv).clamp(-cfg.clip_eps, cfg.clip_eps)
        vl = 0.5 * torch.max((v - br) ** 2, (v_clip - br) ** 2).mean()
        ent = -(logp_all.exp() * logp_all).sum(-1).mean()
        loss = pg + cfg.vf_coef * vl - cfg.ent_coef * ent
        loss.backward()
        stats_s.copy_(torch.stack([loss.detach(), pg.detach(), vl.detach(), ent.detach()]))

    def mb_opt():
        if learner is not None:   # clip + Adam, the ranks' gradient sum averaged inside
            learner.clip_adam(lr_t, cfg.max_grad_norm, 1.0 / world)
            return
        if world > 1:
            flat_grad.div_(world)   # the all-reduce summed the ranks' gradients
        torch.nn.utils.clip_grad_norm_(params, cfg.max_grad_norm, foreach=True)
        opt.step()

    def mb_grad():
        if opt is not None:   # (the manual learner writes every gradient element)
            opt.zero_grad(set_to_none=False)   # the .grad views of flat_grad stay
        mb_step()

    def update_epochs(g_grad=None, g_opt=None):
        """One update; with world > 1 each minibatch is grad graph ->
        all-reduce -> optimizer graph (or the eager calls before capture)."""
        stats_acc.zero_()
        for _ in range(cfg.update_epochs):
            perm = torch.rand(batch_size, device=dev).argsort()   # on the device (randperm builds it on the host)
            for k in range(cfg.n_minibatches):
                idx_s.copy_(perm[k * mb:(k + 1) * mb])
                if g_grad is not None:
                    g_grad.replay()
                else:
                    mb_grad()
                if world > 1:
                    dist.all_reduce(flat_grad)
                if g_opt is not None:
                    g_opt.replay()
                else:
                    mb_opt()
                stats_acc.add_(stats_s)

    g_roll, g_gae, g_upd, g_grad, g_opt = None, None, None, None, None
    pool = None

    def capture(fn, *args):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, pool=pool):
            fn(*args)
        return g

    env.reset()
    history = []
    last_ep, last_ret = 0, 0.0
    t0 = time.perf_counter()
    steps_done = 0
    side = torch.cuda.Stream(device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for upd in range(n_updates):
        ev[0].record()
        if cfg.anneal_lr:
            lr_t.fill_(cfg.lr * (1.0 - upd / n_updates))
        # --- rollout ---------------------------------------------------------
        with torch.no_grad():
            refresh_roll_w()
            for t in range(T + 1):
                if g_roll is None:
                    roll_step(t)
                else:
                    g_roll[t].replay()
                if t < T:
                    env.step(gb.actions)
            if g_gae is None:
                gae_step()
            else:
                g_gae.replay()
        ev[1].record()
        # --- update ----------------------------------------------------------
        if g_upd is not None:
            g_upd.replay()
        elif g_grad is not None:
            update_epochs(g_grad, g_opt)
        else:   # update 0 runs eagerly (warming autograd / cuBLAS / Adam state up)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                update_epochs()
            torch.cuda.current_stream().wait_stream(side)
        if g_roll is None:   # after the eager warm-up update: capture the rollout and GAE
            torch.cuda.synchronize()
            with torch.no_grad():
                # the pre-cast rollout forward is the module's forward
                refresh_roll_w()
                la, va = roll_policy(buf_obs[0])
                lb, vb = policy(buf_obs[0])
                err = max(float((la - lb).abs().max()), float((va - vb).abs().max()))
                assert err < 5e-2, f"rollout forward differs from the module forward by {err}"
                pool = torch.cuda.graph_pool_handle() if pool is None else pool
                g_roll = [capture(roll_step, t) for t in range(T + 1)]
                g_gae = capture(gae_step)
            # the whole update (4 epochs x 8 minibatches: permutation, gather,
            # objective, backward, clip, Adam) as one graph; the gradients stay
            # the tensors the eager update allocated, zeroed in the graph
            if world == 1:
                g_upd = capture(update_epochs)
            else:
                g_grad = capture(mb_grad)
                g_opt = capture(mb_opt)
        ev[2].record()
        steps_done += batch_size * world
        if upd % 10 == 0 or upd == n_updates - 1:
            torch.cuda.synchronize()
            ms_roll, ms_upd = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
            s = (stats_acc / (cfg.update_epochs * cfg.n_minibatches)).tolist()
            st = env.stats()
            mean_ret = st["total_return"] / max(st["episodes"], 1)
            window = (st["total_return"] - last_ret) / max(st["episodes"] - last_ep, 1)
            last_ep, last_ret = st["episodes"], st["total_return"]
            row = {"update": upd, "env_steps": steps_done, "sps": round(steps_done / (time.perf_counter() - t0), 1),
                   "loss": s[0], "pg_loss": s[1], "v_loss": s[2], "entropy": s[3],
                   "episodes": st["episodes"], "mean_episode_return": mean_ret,
                   "recent_episode_return": window,
                   "ms_rollout": round(ms_roll, 3), "ms_update": round(ms_upd, 3)}
            history.append(row)
            if rank == 0:
                log(json.dumps(row))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = env.stats()
    return {"config": asdict(cfg), "n_gpus": world, "updates": n_updates, "env_steps": steps_done,
            "seconds": round(dt, 3), "sps": round(steps_done / dt, 1), "episodes_rank0": st["episodes"],
            "mean_episode_return_rank0": st["total_return"] / max(st["episodes"], 1), "history": history,
            "param_checksum": float(sum(float(p_.detach().double().sum()) for p_ in params))}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="PPO (Craftax-1B hyper-parameters) on the B200 batch engine")
    for k, v in asdict(PPOConfig()).items():
        if isinstance(v, bool):
            ap.add_argument(f"--{k.replace('_', '-')}", type=lambda s: s.lower() in ("1", "true", "yes"), default=v)
        else:
            ap.add_argument(f"--{k.replace('_', '-')}", type=type(v), default=v)
    ap.add_argument("--max-updates", type=int, default=None)
    ap.add_argument("--out", default=None, help="write the result JSON here")
    ap.add_argument("--gpus", type=int, default=1, help="ranks (one per GPU); >1 outside torchrun re-launches")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        import subprocess
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), "-m", "paper_2402_16801_b200.ppo",
               *(argv if argv is not None else sys.argv[1:])]
        return subprocess.call(cmd, env=env)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus and args.gpus > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")
    kw = {k: getattr(args, k) for k in asdict(PPOConfig())}
    res = train(PPOConfig(**kw), log=lambda s: print(s, file=sys.stderr, flush=True), max_updates=args.max_updates)
    if int(os.environ.get("RANK", "0")) == 0:
        txt = json.dumps({k: v for k, v in res.items() if k != "history"})
        print(txt, flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                json.dump(res, fh, indent=1)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
