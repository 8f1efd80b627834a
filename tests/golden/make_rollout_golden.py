"""Mint rollout-report goldens from the reference (run HERE, where /root/reference exists).

    python tests/golden/make_rollout_golden.py

Runs the unmodified reference's ``gridrogue.bench.run_rollout_report``
(bench.py:67-107) read-only from /root/reference/pkg/src for a few
(tier, n_envs, total_steps, seed) cases with the random policy and writes
``bench_rollout_report.json`` next to this script.  tests/test_gpu.py checks
paper_2402_16801_b200.bench_report.run_rollout_report against it.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [("classic", 16, 3200, 5), ("classic", 64, 64 * 400, 1), ("extended", 32, 6400, 2),
         ("extended", 48, 48 * 250, 7)]


def main() -> None:
    sys.path.insert(0, REF)
    from gridrogue import CLASSIC, EXTENDED
    from gridrogue.bench import run_rollout_report
    tiers = {"classic": CLASSIC, "extended": EXTENDED}
    out = []
    for tier, n, total, seed in CASES:
        rep = run_rollout_report(tiers[tier], n, total, policy="random", seed=seed)
        out.append({"args": [tier, n, total, seed], "report": rep})
        print(tier, n, total, seed, rep["episodes_completed"], rep["mean_return"], flush=True)
    with open(os.path.join(OUT, "bench_rollout_report.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
