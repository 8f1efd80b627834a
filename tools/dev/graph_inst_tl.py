"""Dev: kernel timeline of each re-captured step graph (fast vs slow instantiations).
    PYTHONPATH=. python tools/dev/graph_inst_tl.py [n_envs] [tier]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

from paper_2402_16801_b200 import GridrogueBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
tier = sys.argv[2] if len(sys.argv) > 2 else "extended"
gb = GridrogueBatch(n, tier, 0, "symbolic", newly=False, info=False)
gb.reset()
gb.set_validate(False)
t = 0
for k in range(400):
    gb.random_actions(0, t); gb.step(gb.actions); t += 1
keep = []
for trial in range(6):
    bufs = (torch.empty_like(gb.obs), torch.empty_like(gb.reward), torch.empty_like(gb.done))
    keep.append(bufs)   # distinct addresses: a new graph per trial
    gb.obs, gb.reward, gb.done = bufs
    for k in range(20):
        gb.random_actions(0, t); gb.step(gb.actions); t += 1
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for k in range(6):
            gb.random_actions(0, t); gb.step(gb.actions); t += 1
        torch.cuda.synchronize()
    path = f"/tmp/tl_{os.getpid()}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    st = [i for i, e in enumerate(ev) if "k_random_actions" in e["name"]]
    period = (ev[st[-1]]["ts"] - ev[st[1]]["ts"]) / (len(st) - 2)
    t0 = ev[st[3]]["ts"]
    row = " | ".join(f"{e['name'].split('(')[0].split('::')[-1][:14]} {e['ts'] - t0:.0f}-{e['ts'] + e['dur'] - t0:.0f} s{e['args'].get('stream')}"
                     for e in ev[st[3]:st[4]])
    print(f"trial {trial}: period {period:.1f} us :: {row}")
    os.remove(path)
