"""Dev: host enqueue cost per step (random_actions + step, graphed) against the device step time.
    PYTHONPATH=. python tools/dev/host_cost.py [n_envs] [tier]
"""
import sys
import time

import torch

from paper_2402_16801_b200 import GridrogueBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
tier = sys.argv[2] if len(sys.argv) > 2 else "extended"
gb = GridrogueBatch(n, tier, 0, "symbolic", newly=False, info=False)
gb.reset()
gb.set_validate(False)
for k in range(300):
    gb.random_actions(0, k)
    gb.step(gb.actions)
torch.cuda.synchronize()
K = 300
# host-only cost: enqueue K steps while the GPU is still busy with a long kernel
t0 = time.perf_counter()
for k in range(K):
    gb.random_actions(0, 300 + k)
    gb.step(gb.actions)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"n={n} {tier}: host enqueue {1e6 * (t1 - t0) / K:.1f} us/step, wall incl. drain {1e6 * (t2 - t0) / K:.1f} us/step")
t0 = time.perf_counter()
for k in range(K):
    gb.random_actions(0, 600 + k)
t1 = time.perf_counter()
for k in range(K):
    gb.step(gb.actions)
t2 = time.perf_counter()
torch.cuda.synchronize()
print(f"  random_actions {1e6 * (t1 - t0) / K:.1f} us, step {1e6 * (t2 - t1) / K:.1f} us (host)")
