#!/usr/bin/env python
"""Benchmark: auto-resetting batched env.step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json north star): Craftax-Symbolic (the extended
9-floor tier) with symbolic observations, 65,536 envs per GPU, random policy
(policies.RandomPolicy, generated on device), auto-reset with the optimistic
world pool (reset_ratio 16).  One step = BatchEnv.step semantics: game logic
for every env, pool world generation + install for finished envs, post-reset
observation for every env.  Synthetic: worlds are procedurally generated
from seed 0; there is no dataset.

`value` is device-timed (CUDA events on the stream, barrier + synchronize
on both sides, max over ranks) with state and observations resident in HBM;
one-shard steps replay as a CUDA graph.  The per-kernel breakdown behind
`roofline` comes from a second timed pass over the same number of steps
with a CUDA event pair around every launch (kernel-by-kernel, no graph;
`roofline.profiled_ms_per_step`);
`e2e` is the same metric through the host-buffer C-ABI call (gr_step_host):
H2D of the step's actions and D2H of obs/reward/done/info inside the timed
region.  Symbolic obs go into a gr_host_obs_attach'ed pinned buffer (the
delta transfer: only the words changed since the buffer's last step cross
PCIe and are rewritten on the host); `e2e.dense` is the plain 2.17 GB copy.  State (~2.8 GB) and the per-step obs (2.17 GB) exceed the 126 MB L2,
so no explicit flush is needed between steps.

--impl reference times the reference algorithm on the host CPU cores (the
C oracle port in oracle/, all threads) on the same workload, time-capped.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env-steps/sec (random policy, auto-reset)"
UNIT = "env-steps/s"
SEED = 0
# algorithmic bytes per extended-symbolic env-step:
# 2*S_active (456) + view window (99 + 255) + obs (33,072) + IO (9) + R_amort (232)
STEP_BYTES = {("extended", "symbolic"): 34579, ("classic", "symbolic"): 6281,
              ("extended", "pixels"): 44407, ("classic", "pixels"): 12808,
              ("extended", "none"): 1507, ("classic", "none"): 901}
# dominant kernel (the observation writer): bytes per env per launch.
# symbolic: row written + block/item view window read + 64 B of the
# descriptor; pixels (k_pixels, after k_pixprep): frame written + the 848 /
# 560 B per-env scratch read
OBS_KERNEL_BYTES = {("extended", "symbolic"): 33072 + 99 + 255 + 64,
                    ("classic", "symbolic"): 5380 + 63 + 64,
                    ("extended", "pixels"): 42900 + 848,
                    ("classic", "pixels"): 11907 + 560}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peak_hbm() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(tier: str, obs: str, n_envs: int, budget_s: float = 15.0, tile_px=None,
                 max_episode_length=None, steps: int | None = None, warmup: int = 0) -> dict:
    """The oracle port on the host cores (BatchEnv semantics): ``warmup``
    untimed steps, then ``steps`` timed steps -- or, without ``steps``, as
    many as fit in ``budget_s`` (a bounded sample); the timed loop also stops
    at ``budget_s`` so a run always ends in minutes."""
    import numpy as np
    import oracle as O
    threads = os.cpu_count() or 1
    t0 = time.time()
    b = O.OracleBatch(tier, n_envs, SEED, threads=threads, max_episode_length=max_episode_length or 0)
    init_s = time.time() - t0
    na = O.TIERS[tier]["NA"]
    px = tile_px or (7 if tier == "classic" else 10)

    def one(t):
        b.step(O.random_actions(SEED, t, n_envs, na))
        if obs == "symbolic":
            b.state.encode_symbolic()
        elif obs == "pixels":
            b.state.render_pixels(px)

    t = 0
    for _ in range(warmup):
        one(t)
        t += 1
    done = 0
    t0 = time.time()
    while steps is None or done < steps:
        one(t)
        t += 1
        done += 1
        if time.time() - t0 > budget_s:
            break
    dt = time.time() - t0
    cap = f"{done} of {steps} steps" if steps is not None else f"{done} steps (time-capped {budget_s:.0f} s)"
    return {"value": done * n_envs / dt, "unit": UNIT, "cores": threads, "kind": "port", "steps": done,
            "sample": f"{tier}/{obs}, {n_envs} envs x {cap} after {warmup} warm-up steps and a {init_s:.1f} s "
                      f"batch_reset; oracle/ C port of the reference, OpenMP over envs"}


def run_reference(args, world: int, rank: int):
    if rank != 0:
        return
    # the requested K steps after W warm-up steps, on all host cores; the
    # timed loop stops early at GR_REF_BUDGET_S (default 180 s)
    budget = float(os.environ.get("GR_REF_BUDGET_S", "180"))
    cb = cpu_baseline(args.tier, args.obs, args.envs, budget, args.tile_px, args.max_episode_length,
                      steps=args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": cb["steps"], "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (procedural worlds, seed 0)",
            "config": workload_config(args, world),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    name = {"extended": "Craftax", "classic": "Craftax-Classic"}[args.tier]
    extra = ""
    if args.obs == "pixels":
        extra += f", tile_px {args.tile_px or (7 if args.tier == 'classic' else 10)}"
    if args.max_episode_length:
        extra += f", max_episode_length {args.max_episode_length}"
    return {"workload": f"{name}-{args.obs.capitalize()} random-action rollout with auto-reset "
                        f"({args.envs} envs per GPU, reset_ratio 16{extra}, {args.obs} obs post-reset)",
            "tier": args.tier, "obs": args.obs, "n_envs_per_gpu": args.envs,
            "tile_px": args.tile_px if args.obs == "pixels" else None,
            "max_episode_length": args.max_episode_length,
            "global_envs": args.envs * world, "seed": SEED,
            "l2_policy": "no flush: per-step state+obs (>4.9 GB/GPU) exceed the 126 MB L2",
            "parallelism": f"dp{world} (contiguous env shards, NCCL all-gather of a 16 B record/step)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=65536, help="envs per GPU")
    ap.add_argument("--tier", default="extended", choices=["extended", "classic"])
    ap.add_argument("--obs", default="symbolic", choices=["symbolic", "pixels", "none"])
    ap.add_argument("--tile-px", type=int, default=None, help="pixels: tile size (default 7 classic, 10 extended)")
    ap.add_argument("--max-episode-length", type=int, default=None,
                    help="BatchConfig.max_episode_length (reset stress: 16 or 32, SURVEY.md 8(d) config 4)")
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")

    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import numpy as np
    import torch
    # GR_BENCH_BACKEND=gloo lets a dev run put several ranks on one GPU to
    # exercise the multi-rank path; the measured configuration is NCCL, one GPU per rank
    backend = os.environ.get("GR_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    from paper_2402_16801_b200 import GridrogueBatch, ShardedBatch
    from paper_2402_16801_b200.policies import RandomPolicy

    if world > 1:
        env = ShardedBatch(args.envs * world, args.tier, SEED, args.obs, max_episode_length=args.max_episode_length,
                           tile_px=args.tile_px)
        gb = env.batch
    else:
        env = gb = GridrogueBatch(args.envs, args.tier, SEED, args.obs, max_episode_length=args.max_episode_length,
                                  tile_px=args.tile_px, newly=False, info=False)
    gb.set_validate(False)   # actions come from the device policy: valid by construction
    stream = torch.cuda.current_stream()

    t0 = time.time()
    env.reset()
    torch.cuda.synchronize()
    log(f"[rank {rank}] reset of {gb.n} envs: {time.time() - t0:.2f} s")
    t = 0
    for _ in range(args.warmup):
        gb.random_actions(SEED, t)
        env.step(gb.actions)
        t += 1
    torch.cuda.synchronize()
    gb.kernel_times()   # drop warm-up events

    def timed_steps(k, t):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(k):
            gb.random_actions(SEED, t)
            env.step(gb.actions)
            t += 1
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return ev0.elapsed_time(ev1), t

    # pass 1, the measurement: one-shard steps replay as a CUDA graph, no
    # per-kernel events
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    episodes0 = gb.episodes_completed()
    launches0 = gb.kernel_launches()
    ms, t = timed_steps(args.steps, t)
    launches = gb.kernel_launches() - launches0
    resets_per_step = (gb.episodes_completed() - episodes0) / args.steps
    clk = clocks.stop()
    # pass 2, the per-kernel breakdown behind the roofline: the same steps
    # again with a CUDA event pair around every launch (kernel-by-kernel
    # launches, no graph), timed the same way
    gb.set_profiling(True)
    ms_prof, t = timed_steps(args.steps, t)
    gb.set_profiling(False)
    ktimes = gb.kernel_times()
    if dist:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = args.envs * world * args.steps / (ms / 1000.0)

    # roofline of the dominant kernel (device-ms share of the step)
    peak, peak_src = peak_hbm()
    dom = max(ktimes, key=lambda k: ktimes[k][0])
    dom_ms, dom_n = ktimes[dom]
    key = (args.tier, args.obs)
    if dom == "obs" and key in OBS_KERNEL_BYTES:
        # the main writer renders every env not reset this step; the reset
        # envs are rendered by a small launch after their install (obs_reset)
        bytes_per_launch = int(OBS_KERNEL_BYTES[key] * (gb.n - resets_per_step))
    else:
        bytes_per_launch = STEP_BYTES[key] * gb.n
    per_launch_ms = dom_ms / max(dom_n, 1)
    achieved = bytes_per_launch / (per_launch_ms / 1000.0) / 1e9 if per_launch_ms > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        traffic = tr.get(f"{args.tier}_{args.obs}_{dom}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "bytes_per_launch": bytes_per_launch, "ms_per_launch": round(per_launch_ms, 5),
                "share_of_step": round(dom_ms / ms_prof, 3), "peak_source": peak_src,
                "profiled_ms_per_step": round(ms_prof / args.steps, 5),
                "resets_per_step": round(resets_per_step, 1),
                "step_frac": round(value / world * STEP_BYTES[key] / 1e9 / peak, 4)}

    # end to end through the host-buffer C ABI (pinned host memory)
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, gb, env, world, rank, dist, t)

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.tier, args.obs, args.envs, float(os.environ.get("GR_CPU_BUDGET_S", "15")),
                              args.tile_px, args.max_episode_length)
        except Exception as ex:   # the oracle is only the reported baseline
            cb = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (procedural worlds, seed 0; random policy)",
                "config": workload_config(args, world), "roofline": roofline,
                "cpu_baseline": cb, "e2e": e2e, "clocks": clk, "gpu_launches": int(launches),
                "kernel_ms": {k: round(v[0], 3) for k, v in ktimes.items()},
                "worldgen": gb.worldgen_counters()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_e2e(args, gb, env, world, rank, dist, t):
    import numpy as np
    import torch
    from paper_2402_16801_b200 import _lib
    from paper_2402_16801_b200.policies import RandomPolicy
    import ctypes
    n = gb.n
    pol = RandomPolicy(SEED, gb.n_actions)
    acts = [pol.actions_at(t + k, n, env0=gb.cfg.env_offset) for k in range(args.e2e_steps)]
    h_act = torch.empty(n, dtype=torch.int64, pin_memory=True)
    h_obs = torch.empty(tuple(gb.obs.shape), dtype=gb.obs.dtype, pin_memory=True)
    h_rew = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_done = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_newly = torch.empty((n, gb.n_achievements), dtype=torch.uint8, pin_memory=True)
    h_time = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_floor = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    P = lambda x: ctypes.c_void_p(x.data_ptr())
    obs_p = P(h_obs) if args.obs != "none" else None
    d2h = h_obs.numel() * h_obs.element_size() + n * (4 + 1 + gb.n_achievements + 4 + 1)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    if world == 1:
        def host_steps():
            # one warm-up call allocates the library's host-path scratch
            h_act.numpy()[:] = acts[0]
            _lib.check(_lib.lib().gr_step_host(gb.h, P(h_act), obs_p, P(h_rew), P(h_done), P(h_newly),
                                               P(h_time), P(h_floor)))
            t0 = time.perf_counter()
            for k in range(1, args.e2e_steps):
                h_act.numpy()[:] = acts[k]
                _lib.check(_lib.lib().gr_step_host(gb.h, P(h_act), obs_p, P(h_rew), P(h_done), P(h_newly),
                                                   P(h_time), P(h_floor)))
            return time.perf_counter() - t0

        dt = host_steps()
        steps = args.e2e_steps - 1
        if args.obs == "symbolic" and n * h_obs.shape[1] < 2 ** 32:
            # the same calls into an attached buffer (BatchEnv(obs_transfer="delta")):
            # only the obs words that changed since the buffer's last step cross PCIe
            dense = {"value": round(n * steps / dt, 1), "unit": UNIT, "h2d_bytes_per_step": n * 8,
                     "d2h_bytes_per_step": int(d2h), "steps": steps, "path": "gr_step_host, dense obs copy"}
            _lib.check(_lib.lib().gr_host_obs_attach(gb.h, obs_p))
            dt = host_steps()
            prev = h_obs.numpy().view(np.uint32).copy()
            h_act.numpy()[:] = acts[0]
            _lib.check(_lib.lib().gr_step_host(gb.h, P(h_act), obs_p, P(h_rew), P(h_done), P(h_newly),
                                               P(h_time), P(h_floor)))
            changed = int(np.count_nonzero(h_obs.numpy().view(np.uint32) != prev))   # one step's list length
            _lib.check(_lib.lib().gr_host_obs_detach(gb.h, obs_p))
            d2h_delta = 2 * 8 + changed * 8 + n * (4 + 1 + gb.n_achievements + 4 + 1)
            return {"value": round(n * steps / dt, 1), "unit": UNIT, "h2d_bytes_per_step": n * 8,
                    "d2h_bytes_per_step": int(d2h_delta), "steps": steps,
                    "path": "gr_step_host into a gr_host_obs_attach'ed pinned buffer (BatchEnv obs_transfer='delta'): "
                            "(index, value) of the obs words changed since the buffer's last step, host scatter",
                    "dense": dense}
    else:
        d_act = torch.empty(n, dtype=torch.int64, device=gb.device)
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            h_act.numpy()[:] = acts[k]
            d_act.copy_(h_act, non_blocking=True)
            obs, rew, done, newly, tm, fl = env.step(d_act)
            h_obs.copy_(obs, non_blocking=True)
            h_rew.copy_(rew, non_blocking=True)
            h_done.copy_(done, non_blocking=True)
            h_newly.copy_(newly, non_blocking=True)
            h_time.copy_(tm, non_blocking=True)
            h_floor.copy_(fl, non_blocking=True)
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        steps = args.e2e_steps
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    return {"value": round(n * world * steps / dt, 1), "unit": UNIT, "h2d_bytes_per_step": n * 8,
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "path": "gr_step_host (C ABI, pinned host buffers)" if world == 1 else
                    "ShardedBatch.step + pinned H2D/D2H copies"}


if __name__ == "__main__":
    main()
