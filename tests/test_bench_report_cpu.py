"""Host logic of the bench clone (paper_2402_16801_b200.bench_report), no GPU.

The achievement table and the report assembly are checked against the
reference's own rollout reports (tests/golden/bench_rollout_report.json, minted
by tests/golden/make_rollout_golden.py from gridrogue.bench).
"""

import json
import os

import numpy as np
import pytest

from paper_2402_16801_b200 import achievements as A
from paper_2402_16801_b200 import bench_report as B

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bench_rollout_report.json")


def _gold():
    with open(GOLD) as fh:
        return json.load(fh)


def test_achievement_names_and_max_return_match_reference_reports():
    for g in _gold():
        tier = g["args"][0]
        rep = g["report"]
        assert list(rep["achievement_rates"]) == list(A.names(tier))
        assert rep["max_return"] == A.max_return(tier) == B.max_return(tier)
    assert A.max_return("extended") == 226.0 and A.max_return("classic") == 22.0


def test_make_report_layout_and_arithmetic():
    n, steps = 4, 100
    stats = {"episodes": 6, "total_return": 9.5, "ach_episodes": np.arange(22)}
    live = np.ones(22, np.int64)
    rep = B.make_report("classic", "random", 3, n, steps, stats, live, 0.5)
    assert rep["total_steps"] == 400 and rep["episodes_counted"] == 10
    assert rep["mean_return"] == pytest.approx(1.0)
    assert rep["return_pct_of_max"] == pytest.approx(100 * 1.0 / 22.0)
    assert rep["achievement_rates"]["COLLECT_WOOD"] == pytest.approx(0.1)
    assert rep["achievement_rates"]["MAKE_IRON_SWORD"] == pytest.approx(2.2)
    assert list(rep) == list(_gold()[0]["report"])


def test_policy_and_argument_errors():
    with pytest.raises(NotImplementedError):
        B.run_rollout_report("classic", 4, 400, policy="scripted")
    with pytest.raises(ValueError):
        B.run_rollout_report("classic", 8, 4)
    with pytest.raises(ValueError):
        B.run_speed_sweep("classic", [], 100)
    with pytest.raises(ValueError):
        B.make_report("nope", "random", 0, 1, 1, {"episodes": 0, "total_return": 0, "ach_episodes": []}, [], 0)
