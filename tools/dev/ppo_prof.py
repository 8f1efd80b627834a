"""Dev: kernel-time table of the graphed PPO loop (torch.profiler; not a bench number)."""
import sys
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2402_16801_b200.ppo import PPOConfig, train

cfg = PPOConfig(total_timesteps=1024 * 64 * 6)
train(cfg, log=lambda s: None, max_updates=3)   # warm (captures happen in update 0)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    train(cfg, log=lambda s: None, max_updates=4)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=int(sys.argv[1]) if len(sys.argv) > 1 else 30))
