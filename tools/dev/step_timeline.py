"""Dev: kernel timeline (start / duration / stream) of steady-state graphed
steps of the bench workload, from a torch.profiler trace (not a bench number).
    PYTHONPATH=. python tools/dev/step_timeline.py [n_envs] [obs]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2402_16801_b200 import GridrogueBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
obs = sys.argv[2] if len(sys.argv) > 2 else "symbolic"
gb = GridrogueBatch(n, "extended", 0, obs, newly=False, info=False)
gb.reset()
gb.set_validate(False)
for k in range(400):
    gb.random_actions(0, k)
    gb.step(gb.actions)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(400, 406):
        gb.random_actions(0, k)
        gb.step(gb.actions)
    torch.cuda.synchronize()
path = "gpurun_out/step_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
st = [i for i, e in enumerate(ev) if "k_random_actions" in e["name"]]
t0 = ev[st[2]]["ts"]
for e in ev[st[2]: st[4]]:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  end {e['ts'] + e['dur'] - t0:9.1f}  s{e['args'].get('stream')}  "
          f"{e['name'][:80]}")
os.remove(path)
