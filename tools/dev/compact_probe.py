"""dev probe: gr_obs_to_host (compact transfer) vs n, destination kind."""
import sys, time, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2402_16801_b200 import GridrogueBatch
for n in (4096, 16384, 65536):
    gb = GridrogueBatch(n, "extended", 0, "symbolic")
    gb.reset()
    for kind in ("pinned", "numpy"):
        out = torch.empty(tuple(gb.obs.shape), dtype=torch.float32, pin_memory=True).numpy() if kind == "pinned" else np.zeros(tuple(gb.obs.shape), np.float32)
        gb.obs_to_host(out)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter(); gb.obs_to_host(out); ts.append(time.perf_counter() - t0)
        print(n, kind, "ms", [round(1e3 * t, 2) for t in ts], "GB/s", round(out.nbytes / min(ts) / 1e9, 1), flush=True)
    del gb
