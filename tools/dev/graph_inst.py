"""Dev: is the step schedule decided per graph instantiation or per process?
Re-captures the step graph with fresh output buffers several times in one
process and times each.
    PYTHONPATH=. python tools/dev/graph_inst.py [n_envs] [tier]
"""
import sys

import torch

from paper_2402_16801_b200 import GridrogueBatch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
tier = sys.argv[2] if len(sys.argv) > 2 else "classic"
gb = GridrogueBatch(n, tier, 0, "symbolic", newly=False, info=False)
gb.reset()
gb.set_validate(False)
t = 0
for k in range(400):
    gb.random_actions(0, t); gb.step(gb.actions); t += 1
out = []
for trial in range(8):
    gb.obs = torch.empty_like(gb.obs)
    gb.reward = torch.empty_like(gb.reward)
    gb.done = torch.empty_like(gb.done)
    for k in range(30):
        gb.random_actions(0, t); gb.step(gb.actions); t += 1
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(300):
        gb.random_actions(0, t); gb.step(gb.actions); t += 1
    e1.record()
    torch.cuda.synchronize()
    out.append(round(e0.elapsed_time(e1) / 300, 4))
print(n, tier, "ms/step per re-captured graph:", out)
