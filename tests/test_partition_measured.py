"""Partitioning driven by measured stage periods.

CPU: with the simulated period oracle the Python search reproduces the native partitioner
(the reference's Algorithm 1) exactly — same layers, durations, moves. GPU: with B200-timed
stage periods (standalone stage executors) the search runs and returns a valid partition.
"""
import json
from fractions import Fraction

import pytest

from paper_2406_08756_b200 import gpt_profile as gp
from paper_2406_08756_b200 import partition_measured as pm
from paper_2406_08756_b200 import planner


@pytest.mark.parametrize("key,budget", [("1.3b", None), ("7b", None), ("13b", 40_000_000_000), ("1.3b", 24_000_000_000)])
def test_search_with_simulated_periods_matches_native(key, budget):
    c = gp.CONFIGS[key]
    if budget:
        c = gp.GPTConfig(**{**c.__dict__, "mem_budget_bytes": budget})
    text = gp.profile_text(c)
    native = json.loads(planner.partition_text(text))
    mine = pm.search_partition(text, pm.simulated_period(text))
    assert mine["layers_per_stage"] == native["layers_per_stage"]
    assert mine["iterations"] == native["iterations"]
    assert [(m["from"], m["to"]) for m in mine["moves"]] == [(m["from"], m["to"]) for m in native["moves"]]
    for a, b in zip(mine["durations_us"], native["durations_us"]):
        assert abs(Fraction(a) - Fraction(b)) < Fraction(1, 1000)  # native prints 3 decimals


@pytest.mark.gpu
def test_search_with_measured_periods(cuda):
    c = gp.GPTConfig("gpt-tiny-pp", 8, 512, 8, 256, 2, 50304, 1, 2, 4, dropout=0.1)
    text = gp.profile_text(c)
    part = pm.search_partition(text, pm.measured_period(c, text, steps=1, warmup=1))
    assert sum(part["layers_per_stage"]) == c.n_layers and all(x >= 1 for x in part["layers_per_stage"])
    assert all(Fraction(d) > 0 for d in part["durations_us"])
    assert len(part["measured"]) >= 2
