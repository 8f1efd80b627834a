"""Dev: kernel-time table of the graphed PPO loop (torch.profiler; not a bench number)."""
import sys
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2402_16801_b200.ppo import PPOConfig, train

cfg = PPOConfig(total_timesteps=1024 * 64 * 6)
train(cfg, log=lambda s: None, max_updates=3)   # warm (captures happen in update 0)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    train(cfg, log=lambda s: None, max_updates=4)
rows = [(e.key, e.device_time_total, e.count) for e in prof.key_averages()]
rows.sort(key=lambda r: -r[1])
tot = sum(r[1] for r in rows)
for k, t, c in rows[: int(sys.argv[1]) if len(sys.argv) > 1 else 40]:
    print(f"{t / 1e3:9.2f} ms {t / tot:6.3f} {c:7d}  {k[:160]}")
