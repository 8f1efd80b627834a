"""Dev: kernel timeline of graphed steady-state steps (torch.profiler), with
the mean step period, to compare schedules across processes.
    PYTHONPATH=. python tools/dev/step_timeline2.py [n_envs]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2402_16801_b200 import GridrogueBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
gb = GridrogueBatch(n, "extended", 0, "symbolic", newly=False, info=False)
gb.reset()
gb.set_validate(False)
for k in range(400):
    gb.random_actions(0, k)
    gb.step(gb.actions)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(400, 420):
        gb.random_actions(0, k)
        gb.step(gb.actions)
    torch.cuda.synchronize()
path = f"/tmp/step_trace_{os.getpid()}.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
st = [i for i, e in enumerate(ev) if "k_random_actions" in e["name"]]
period = (ev[st[-1]]["ts"] - ev[st[2]]["ts"]) / (len(st) - 3)
print(f"period {period:.1f} us")
t0 = ev[st[10]]["ts"]
for e in ev[st[10]: st[11]]:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  end {e['ts'] + e['dur'] - t0:9.1f}  s{e['args'].get('stream')}  {e['name'][:60]}")
os.remove(path)
