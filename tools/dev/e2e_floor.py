"""Dev: where the host path's time goes at small batches (not a bench number).

Per size: the device-timed graph step, gr_step_host without an observation,
BatchEnv.step (dense, writable arrays) with gr_host_phase_times.
    PYTHONPATH=. python tools/dev/e2e_floor.py [n ...]
"""
import ctypes
import sys
import time

import numpy as np
import torch

from paper_2402_16801_b200 import BatchEnv, GridrogueBatch
from paper_2402_16801_b200._lib import check, lib
from paper_2402_16801_b200.policies import RandomPolicy


def phases(gb):
    ms = (ctypes.c_double * 4)()
    calls, words = ctypes.c_int64(), ctypes.c_int64()
    check(lib().gr_host_phase_times(gb.h, ms, ctypes.byref(calls), ctypes.byref(words)))
    return [round(x / max(calls.value, 1), 4) for x in ms], calls.value


for n in [int(x) for x in sys.argv[1:]] or [1024, 4096, 16384]:
    gb = GridrogueBatch(n, "extended", 0, "symbolic")
    gb.reset()
    pol = RandomPolicy(0, gb.n_actions)
    acts = [pol.actions_at(k, n) for k in range(64)]
    dacts = [torch.from_numpy(a).cuda() for a in acts]
    for k in range(200):
        gb.step(dacts[k % 64])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(200):
        gb.step(dacts[k % 64])
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / 200
    # host path without an observation
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    ha, hr, hd = pin(n, torch.int64), pin(n, torch.float32), pin(n, torch.bool)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    for k in range(20):
        ha[:] = acts[k % 64]
        check(lib().gr_step_host(gb.h, vp(ha), None, vp(hr), vp(hd), None, None, None))
    phases(gb)
    t0 = time.perf_counter()
    for k in range(200):
        ha[:] = acts[k % 64]
        check(lib().gr_step_host(gb.h, vp(ha), None, vp(hr), vp(hd), None, None, None))
    noobs_ms = (time.perf_counter() - t0) * 1e3 / 200
    ph_noobs = phases(gb)
    env = BatchEnv.from_batch(gb, "dense")
    for k in range(20):
        o, r, d, i = env.step(acts[k % 64])
        del o, r, d, i
    phases(gb)
    t0 = time.perf_counter()
    for k in range(100):
        o, r, d, i = env.step(acts[k % 64])
        del o, r, d, i
    be_ms = (time.perf_counter() - t0) * 1e3 / 100
    ph_be = phases(gb)
    print(f"n={n}: device {dev_ms:.4f} ms | step_host no obs {noobs_ms:.4f} ms {ph_noobs} | "
          f"BatchEnv dense {be_ms:.4f} ms {ph_be} -> {n / be_ms * 1e3 / 1e6:.2f} M/s", flush=True)
    env.close()
    del env, gb
