"""A short two-stream rollout for compute-sanitizer (race detection).

    compute-sanitizer --tool memcheck  python tools/sanitize_rollout.py
    compute-sanitizer --tool racecheck python tools/sanitize_rollout.py
    compute-sanitizer --tool synccheck python tools/sanitize_rollout.py
    compute-sanitizer --tool initcheck python tools/sanitize_rollout.py

Extended tier, symbolic and pixel observations, reset stress
(max_episode_length 12, so every step runs the reset chain -- compaction,
worldgen, install, reset-env obs -- on the side stream beside the main
observation writer), the sharded halves (gr_step_local / gr_step_finish) and
the delta host transfer; kernel-by-kernel launches (GR_GRAPH=0) and the
captured-graph path both run.  Small batches keep the sanitizer's replay
time in minutes.
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2402_16801_b200 import BatchEnv, GridrogueBatch
    steps = int(os.environ.get("GR_SAN_STEPS", "50"))
    for tier, obs, n in (("extended", "symbolic", 512), ("extended", "pixels", 64), ("classic", "symbolic", 256)):
        gb = GridrogueBatch(n, tier, 3, obs, max_episode_length=12)
        gb.reset()
        gb.set_validate(False)
        for t in range(steps):
            gb.random_actions(3, t)
            gb.step(gb.actions)
        torch.cuda.synchronize()
        ex = torch.zeros(4, dtype=torch.int32, device="cuda")
        for t in range(steps, steps + 5):   # the sharded halves (world size 1)
            gb.random_actions(3, t)
            gb.step_local(gb.actions, ex)
            gb.step_finish(ex, 0, 1)
        torch.cuda.synchronize()
        print(f"{tier}/{obs}: {steps + 5} steps, {gb.episodes_completed()} episodes", flush=True)
    env = BatchEnv(256, "extended", 5, "symbolic", max_episode_length=12, obs_transfer="delta")
    env.reset()
    rng = np.random.default_rng(0)
    for _ in range(20):
        obs, rew, done, info = env.step(rng.integers(0, env.n_actions, 256))
    env.close()
    print("delta transfer: 20 steps", flush=True)


if __name__ == "__main__":
    main()
