"""Dev: kernel timeline (start / end per stream) of a few graphed PPO rollout
steps and one minibatch, from a torch.profiler chrome trace (not a bench number).
    PYTHONPATH=. python tools/dev/ppo_timeline.py
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2402_16801_b200.ppo import PPOConfig, train

cfg = PPOConfig(total_timesteps=1024 * 64 * 3)
train(cfg, log=lambda s: None, max_updates=2)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    train(cfg, log=lambda s: None, max_updates=3)
path = "gpurun_out/ppo_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
# the last update's rollout: find the k_step launches, show 3 steps around the middle
steps = [i for i, e in enumerate(ev) if "k_step" in e["name"]]
mid = steps[-40]
t0 = ev[mid]["ts"]
print("rollout steps (us from a k_step start):")
for e in ev[mid - 30: mid + 60]:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  s{e['args'].get('stream')}  {e['name'][:90]}")
# one minibatch of the last update: between two k_adam launches
ad = [i for i, e in enumerate(ev) if "k_adam" in e["name"]]
if len(ad) >= 3:
    a, b = ad[-3], ad[-2]
    t0 = ev[a]["ts"]
    print("\nminibatch (us from a k_adam start):")
    for e in ev[a: b + 1]:
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  s{e['args'].get('stream')}  {e['name'][:90]}")
os.remove(path)
