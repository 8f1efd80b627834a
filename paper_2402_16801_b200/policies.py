"""Host-side action source: policies.RandomPolicy restated in numpy.

Uniform random actions, deterministic in (seed, step, global env index)
(/root/reference/pkg/src/gridrogue/policies.py:22-37).  The device twin is
gr_random_actions; this one feeds the host (end-to-end) path.
"""

from __future__ import annotations

import numpy as np

_G = np.uint32(0x9E3779B9)


def _mix32(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint32(16))
    x = x * np.uint32(0x7FEB352D)
    x = x ^ (x >> np.uint32(15))
    x = x * np.uint32(0x846CA68B)
    return x ^ (x >> np.uint32(16))


class RandomPolicy:
    def __init__(self, seed: int, n_actions: int):
        self.key = int(seed) & 0xFFFFFFFF
        self.n_actions = int(n_actions)
        self.t = 0

    def actions_at(self, t: int, n: int, env0: int = 0) -> np.ndarray:
        k = np.uint32((self.key + t * 2654435761) & 0xFFFFFFFF)
        idx = np.arange(env0, env0 + n, dtype=np.uint32)
        with np.errstate(over="ignore"):
            h = _mix32(k ^ (idx * _G + _G))
        u = (h >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / (1 << 24))
        return (u * np.float32(self.n_actions)).astype(np.int64) % self.n_actions

    def actions(self, n: int, env0: int = 0) -> np.ndarray:
        a = self.actions_at(self.t, n, env0)
        self.t += 1
        return a
