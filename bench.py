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

Both arms first pre-roll ``--preroll`` (default 400, ~2x the mean episode
length) untimed steps from batch_reset so the timed window sees the steady
reset rate (~275 resets/step at 65,536 envs), then W warm-up steps, then K
timed steps; both print ``resets_per_step``.

`value` is device-timed (CUDA events on the stream, barrier + synchronize
on both sides, max over ranks) with state and observations resident in HBM;
steps replay as a CUDA graph (N > 1: local step + NCCL all-gather + finish
captured in one graph).  The per-kernel breakdown behind `roofline` comes
from a second timed pass over the same number of steps with a CUDA event
pair around every launch (kernel-by-kernel, no graph;
`roofline.profiled_ms_per_step`).

`e2e` is the same metric through the reference-facing numpy API,
``BatchEnv.step`` (bindings/src/gridrogue_gym/__init__.py:63-84) on host
arrays: H2D of the actions and D2H of obs / reward / done / info inside the
timed region.  ``e2e.value`` is the reference's contract (writable
observation arrays, a dense 2.17 GB copy per step, PCIe-bound);
``e2e.delta`` is BatchEnv(obs_transfer="delta") (read-only arrays owned by the
handle; only the words changed since a buffer's last step cross PCIe).  Each
carries the host-measured phase breakdown (gr_host_phase_times) and is the
median of three windows of --e2e-steps steps (listed with their spread: the
host-side phases vary with the box's host load).  State
(~2.8 GB) and the per-step obs (2.17 GB) exceed the 126 MB L2, so no explicit
flush is needed between steps.

--impl reference times the reference algorithm on the host CPU cores (the
C oracle port in oracle/, all threads) on the same workload, time-capped.
--gpus N without torchrun re-launches itself under torch.distributed.run.
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
# k_step: bytes per env per launch -- 2 x the current floor's non-map state
# (SURVEY.md 8(d) S_active), the map window, actions / reward / done and the
# 256-byte observation descriptor it writes
STEP_KERNEL_BYTES = {"extended": 2 * 456 + 99 + 255 + 9 + 256, "classic": 2 * 395 + 63 + 9 + 256}
# k_worldgen: the maps of one generated world (blocks + items, all floors)
WORLD_BYTES = {"extended": 2 * 9 * 48 * 48, "classic": 2 * 64 * 64}
# dominant kernel (the observation writer): bytes per env per launch.
# symbolic: row written + block/item view window read + the 256 B
# descriptor (gr_desc.cuh, read whole); pixels (k_pixels, after k_pixprep): frame written + the 848 /
# 560 B per-env scratch read
OBS_KERNEL_BYTES = {("extended", "symbolic"): 33072 + 99 + 255 + 256,
                    ("classic", "symbolic"): 5380 + 63 + 256}


def pixel_class_row_bytes(tier: str, px: int) -> int:
    """Bytes per frame of the compact pixel transfer: one row per row class
    (the writer's row_class, gr_obs.cu: tile rows with / without insets and
    gear bar, each vital bar, blank)."""
    ext = tier == "extended"
    vr, vc, side = (9, 11, 2) if ext else (7, 9, 0)
    inset, ns = max(1, px // 4), (5 if ext else 4)
    bar_h = max(2, (2 * px) // (ns + 1))
    classes = set()
    for y in range((vr + 2) * px):
        if y < vr * px:
            r, iy = divmod(y, px)
            classes.add(r * 4 + (inset <= iy < px - inset) + 2 * (ext and r < 7 and 1 <= iy < px - 1))
        else:
            q = y - vr * px - 1
            classes.add(vr * 4 + (q // bar_h if q >= 0 and q // bar_h < ns and q % bar_h < bar_h - 1 else 5))
    return len(classes) * (vc + side) * px * 3


def obs_kernel_bytes(tier: str, obs: str, tile_px: int | None) -> int:
    """Bytes per env per launch of the observation writer; pixel frames are
    ((view rows + 2) x px) x ((view cols + side panel) x px) x 3 (tiles.py:85-100)."""
    if obs == "symbolic":
        return OBS_KERNEL_BYTES[(tier, obs)]
    ext = tier == "extended"
    px = tile_px or (10 if ext else 7)
    vr, vc, side = (9, 11, 2) if ext else (7, 9, 0)
    return (vr + 2) * px * (vc + side) * px * 3 + (848 if ext else 560)


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
    untimed steps (pre-roll + warm-up), then ``steps`` timed steps -- or,
    without ``steps``, as many as fit in ``budget_s`` (a bounded sample); the
    timed loop also stops at ``budget_s`` so a run always ends in minutes."""
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
    t0 = time.time()
    for _ in range(warmup):
        one(t)
        t += 1
    pre_s = time.time() - t0
    ep0 = b.stats()["episodes"]
    done = 0
    t0 = time.time()
    while steps is None or done < steps:
        one(t)
        t += 1
        done += 1
        if time.time() - t0 > budget_s:
            break
    dt = time.time() - t0
    rps = (b.stats()["episodes"] - ep0) / max(done, 1)
    cap = f"{done} of {steps} steps" if steps is not None else f"{done} steps (time-capped {budget_s:.0f} s)"
    return {"value": done * n_envs / dt, "unit": UNIT, "cores": threads, "kind": "port", "steps": done,
            "resets_per_step": round(rps, 1),
            "sample": f"{tier}/{obs}, {n_envs} envs x {cap} after {warmup} untimed pre-roll + warm-up steps "
                      f"({pre_s:.1f} s) and a {init_s:.1f} s batch_reset; oracle/ C port of the reference, "
                      f"one host thread per core over envs"}


def run_reference(args, world: int, rank: int):
    if rank != 0:
        return
    # the requested K steps after the pre-roll and W warm-up steps, on all
    # host cores; the timed loop stops early at GR_REF_BUDGET_S (default 180 s)
    budget = float(os.environ.get("GR_REF_BUDGET_S", "180"))
    cb = cpu_baseline(args.tier, args.obs, args.envs, budget, args.tile_px, args.max_episode_length,
                      steps=args.steps, warmup=args.preroll + args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": cb["steps"], "warmup": args.warmup, "preroll": args.preroll,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (procedural worlds, seed 0)",
            "config": workload_config(args, world),
            "resets_per_step": cb["resets_per_step"],
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
            "global_envs": args.envs * world, "seed": SEED, "preroll_steps": args.preroll,
            "l2_policy": "no flush: per-step state+obs (>4.9 GB/GPU) exceed the 126 MB L2",
            "parallelism": f"dp{world} (contiguous env shards, NCCL all-gather of a 16 B record/step)"}


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _relaunch(args) -> int:
    """--gpus N outside torchrun: run N ranks, one per GPU, under
    torch.distributed.run (127.0.0.1 rendezvous); rank 0 prints the line."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")   # the communicator's rank count goes to the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    log("launching", " ".join(cmd))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--preroll", type=int, default=400,
                    help="untimed steps from batch_reset before the warm-up (steady-state reset rate)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--envs", type=int, default=65536, help="envs per GPU")
    ap.add_argument("--tier", default="extended", choices=["extended", "classic"])
    ap.add_argument("--obs", default="symbolic", choices=["symbolic", "pixels", "none"])
    ap.add_argument("--tile-px", type=int, default=None, help="pixels: tile size (default 7 classic, 10 extended)")
    ap.add_argument("--max-episode-length", type=int, default=None,
                    help="BatchConfig.max_episode_length (reset stress: 16 or 32, SURVEY.md 8(d) config 4)")
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch / rank / config plumbing only (gloo, no GPU work): prints the config line")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")

    in_torchrun = "WORLD_SIZE" in os.environ
    if args.impl == "ours" and args.gpus > 1 and not in_torchrun:
        if args.dry_run:
            os.environ.setdefault("GR_BENCH_BACKEND", "gloo")
        sys.exit(_relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, max(world, args.gpus), rank)
        return
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.dry_run:
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            assert dist.get_world_size() == args.gpus
            dist.barrier()
            dist.destroy_process_group()
        if rank == 0:
            print(json.dumps({"dry_run": True, "n_gpus": world, "config": workload_config(args, world)}), flush=True)
        return

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
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        assert dist.get_world_size() == args.gpus

    from paper_2402_16801_b200 import GridrogueBatch, ShardedBatch

    if world > 1:
        env = ShardedBatch(args.envs * world, args.tier, SEED, args.obs, max_episode_length=args.max_episode_length,
                           tile_px=args.tile_px, graph=(backend == "nccl"))
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
    t0 = time.time()
    for _ in range(args.preroll + args.warmup):
        gb.random_actions(SEED, t)
        env.step(gb.actions)
        t += 1
    torch.cuda.synchronize()
    log(f"[rank {rank}] pre-roll {args.preroll} + warm-up {args.warmup} steps: {time.time() - t0:.2f} s")
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

    # pass 1, the measurement: steps replay as a CUDA graph, no per-kernel events
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
    ktimes, ms_prof = None, None
    worlds0 = gb.worldgen_counters()["worlds"]
    gb.set_profiling(True)
    if world > 1:   # the same sharded step, launched eagerly so every kernel gets its event pair
        graphed_step, env.step = env.step, env._step_eager
    ms_prof, t = timed_steps(args.steps, t)
    if world > 1:
        env.step = graphed_step
    gb.set_profiling(False)
    ktimes = gb.kernel_times()
    worlds_prof = gb.worldgen_counters()["worlds"] - worlds0
    if dist:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        rr = torch.tensor([resets_per_step], dtype=torch.float64, device="cuda")
        dist.all_reduce(rr)
        resets_per_step = float(rr.item())    # whole job
    value = args.envs * world * args.steps / (ms / 1000.0)

    key = (args.tier, args.obs)
    peak, peak_src = peak_hbm()
    roofline = None
    if ktimes:
        # roofline of the dominant kernel (device-ms share of the step)
        dom = max(ktimes, key=lambda k: ktimes[k][0])
        dom_ms, dom_n = ktimes[dom]
        if dom == "obs" and args.obs in ("symbolic", "pixels"):
            # the main writer renders every env not reset this step; the reset
            # envs are rendered by a small launch after their install (obs_reset)
            bytes_per_launch = int(obs_kernel_bytes(args.tier, args.obs, args.tile_px) * (gb.n - resets_per_step))
        elif dom == "step":
            bytes_per_launch = STEP_KERNEL_BYTES[args.tier] * gb.n
        elif dom == "worldgen":
            # the maps it writes (compute / latency bound: the fraction is small)
            bytes_per_launch = int(WORLD_BYTES[args.tier] * worlds_prof / max(dom_n, 1))
        else:
            bytes_per_launch = STEP_BYTES[key] * gb.n
        per_launch_ms = dom_ms / max(dom_n, 1)
        achieved = bytes_per_launch / (per_launch_ms / 1000.0) / 1e9 if per_launch_ms > 0 else 0.0
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                traffic = json.load(fh).get(f"{args.tier}_{args.obs}_{dom}")
        except Exception:
            pass
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                    "bytes_per_launch": bytes_per_launch, "ms_per_launch": round(per_launch_ms, 5),
                    "share_of_step": round(dom_ms / ms_prof, 3), "peak_source": peak_src,
                    "profiled_ms_per_step": round(ms_prof / args.steps, 5),
                    "resets_per_step": round(resets_per_step, 1),
                    "step_frac": round(value / world * STEP_BYTES[key] / 1e9 / peak, 4)}

    # end to end through the numpy API (pinned host memory)
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, gb, env, world, rank, dist, t)

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.tier, args.obs, args.envs, float(os.environ.get("GR_CPU_BUDGET_S", "15")),
                              args.tile_px, args.max_episode_length, warmup=args.preroll)
        except Exception as ex:   # the oracle is only the reported baseline
            cb = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "preroll": args.preroll,
                "ms_per_step": round(ms / args.steps, 5),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (procedural worlds, seed 0; random policy)",
                "config": workload_config(args, world), "resets_per_step": round(resets_per_step, 1),
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "clocks": clk, "gpu_launches": int(launches),
                "kernel_ms": {k: round(v[0], 3) for k, v in ktimes.items()} if ktimes else None,
                "worldgen": gb.worldgen_counters()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _phases(gb) -> dict:
    import ctypes
    import numpy as np
    from paper_2402_16801_b200 import _lib
    out = np.zeros(4, np.float64)
    calls, words = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().gr_host_phase_times(gb.h, out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(calls),
                                              ctypes.byref(words)))
    c = max(calls.value, 1)
    return {"ms_per_step": {"enqueue": round(out[0] / c, 3), "device_wait": round(out[1] / c, 3),
                            "host_scatter": round(out[2] / c, 3), "final_sync": round(out[3] / c, 3)},
            "changed_words_per_step": int(words.value / c)}   # delta: changed words; compact: non-zero words


E2E_WINDOWS = 3


def run_e2e(args, gb, env, world, rank, dist, t):
    import numpy as np
    import torch
    from paper_2402_16801_b200 import BatchEnv
    from paper_2402_16801_b200.policies import RandomPolicy
    n = gb.n
    pol = RandomPolicy(SEED, gb.n_actions)
    steps = args.e2e_steps
    acts = [pol.actions_at(t + k, n, env0=gb.cfg.env_offset) for k in range(steps * E2E_WINDOWS + 2)]
    small_d2h = n * (4 + 1 + gb.n_achievements + 4 + 1)   # reward, done, newly, time, floor
    obs_bytes = int(np.prod(gb.obs.shape[1:])) * gb.obs.element_size() * n
    # the library's choice for host arrays (gr_create): the compact transfer
    # unless disabled or below GR_HOST_COMPACT_MIN_MB of observations a step
    compact = (os.environ.get("GR_HOST_COMPACT", "1") != "0"
               and obs_bytes / 1048576.0 >= float(os.environ.get("GR_HOST_COMPACT_MIN_MB", "40")))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    if world == 1:
        def run(be, k0):
            # BatchEnv.step is the timed call; the caller drops each step's
            # arrays before the next step, like a training loop would.  Three
            # windows of `steps` steps: the median is reported, the windows
            # beside it (the host-side phases vary with the box's host load)
            be.step(acts[k0])
            _phases(gb)
            vals = []
            for w in range(E2E_WINDOWS):
                t0 = time.perf_counter()
                for k in range(steps):
                    obs, rew, done, info = be.step(acts[k0 + 1 + w * steps + k])
                    del obs, rew, done, info
                vals.append(n * steps / (time.perf_counter() - t0))
            ph = _phases(gb)
            ph["windows"] = [round(v, 1) for v in vals]
            ph["spread"] = round((max(vals) - min(vals)) / statistics.median(vals), 4)
            return statistics.median(vals), ph

        dense_env = BatchEnv.from_batch(gb, "dense")
        v_dense, ph_dense = run(dense_env, 0)
        dense_env.close()
        if args.obs == "symbolic" and compact:
            nb = (gb.obs.shape[1] + 31) // 32
            d2h_dense = n * nb * 4 + n * 8 + ph_dense["changed_words_per_step"] * 4 + small_d2h
            how = ("the observation travels packed (per row a non-zero bitmap + its values, gr_host_phase_times "
                   "words) and host threads expand it into the whole array (AVX-512 expand, streaming stores)")
        elif args.obs == "pixels" and compact:
            d2h_dense = n * pixel_class_row_bytes(args.tier, gb.tile_px) + small_d2h
            how = ("the frames travel as one row per row class (rows of a class are byte-identical) and host "
                   "threads replicate them into the whole array")
        else:
            d2h_dense = obs_bytes + small_d2h
            how = "D2H of the whole observation"
        out = {"value": round(v_dense, 1), "unit": UNIT, "h2d_bytes_per_step": n * 8,
               "d2h_bytes_per_step": int(d2h_dense), "steps": steps,
               "path": "BatchEnv.step (numpy in/out, writable obs arrays as the reference returns): "
                       "H2D actions, device step, " + how + ", D2H of reward/done/info",
               "phases": ph_dense}
        if args.obs == "symbolic" and n * gb.obs.shape[1] < 2 ** 32:
            delta_env = BatchEnv.from_batch(gb, "delta")
            delta_env.step(acts[0])      # first delivery into each buffer is a full one
            delta_env.step(acts[1])
            delta_env.step(acts[0])
            v_delta, ph_delta = run(delta_env, 0)
            delta_env.close()
            out["delta"] = {"value": round(v_delta, 1), "unit": UNIT, "h2d_bytes_per_step": n * 8,
                            "d2h_bytes_per_step": int(ph_delta["changed_words_per_step"] * 8 + small_d2h),
                            "steps": steps,
                            "path": "BatchEnv(obs_transfer='delta').step: read-only obs arrays owned by the handle; "
                                    "(index, value) of the words changed since a buffer's last step, listed on the device "
                                    "in 8 row chunks, each copied back while the next is listed and scattered by host threads",
                            "phases": ph_delta}
        return out
    d_act = torch.empty(n, dtype=torch.int64, device=gb.device)
    h_act = torch.empty(n, dtype=torch.int64, pin_memory=True)
    h_obs = np.empty(tuple(gb.obs.shape), dtype=np.float32 if args.obs == "symbolic" else np.uint8)
    h_small = [torch.empty(tuple(x.shape), dtype=x.dtype, pin_memory=True)
               for x in (gb.reward, gb.done, gb.newly, gb.time, gb.floor)]
    gb.obs_to_host(h_obs)   # first call allocates the transfer's buffers
    _phases(gb)
    t0 = time.perf_counter()
    for k in range(steps):
        h_act.numpy()[:] = acts[k]
        d_act.copy_(h_act, non_blocking=True)
        obs, *rest = env.step(d_act)
        for h, d in zip(h_small, rest):
            h.copy_(d, non_blocking=True)
        gb.obs_to_host(h_obs)   # waits for this step's obs on the current stream
        torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ph = _phases(gb)
    tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt = float(tt.item())
    if args.obs == "symbolic" and compact:
        d2h = n * ((gb.obs.shape[1] + 31) // 32) * 4 + n * 8 + ph["changed_words_per_step"] * 4 + small_d2h
    elif args.obs == "pixels" and compact:
        d2h = n * pixel_class_row_bytes(args.tier, gb.tile_px) + small_d2h
    else:
        d2h = obs_bytes + small_d2h
    return {"value": round(n * world * steps / dt, 1), "unit": UNIT, "h2d_bytes_per_step": n * 8,
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "path": "ShardedBatch.step (local step + all-gather + finish; one CUDA graph with NCCL) + H2D actions, "
                    "GridrogueBatch.obs_to_host (compact transfer into a numpy array), D2H reward/done/info (per rank)",
            "phases": ph}


if __name__ == "__main__":
    main()
