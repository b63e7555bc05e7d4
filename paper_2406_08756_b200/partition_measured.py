"""Pipeline partitioning driven by measured stage periods.

The reference's Algorithm 1 (`search_partition`, proj/src/partition.cpp:111-215; here the
native `host/partition.cpp: greedy_partition`) balances *simulated* stage periods
(`stage_period_us`, pipesim.cpp:767-779). This module runs the same search with a pluggable
period oracle:

    part = search_partition(profile_text, period=measured_period(c))   # B200-timed stages
    part = search_partition(profile_text, period=simulated_period(t))  # == the native result

`measured_period` times one stage alone on one GPU (executor option `standalone_stage`:
pipeline receives read synthetic activations / gradients, sends are skipped) with that
stage's own HEU plan, and reports the iteration time per microbatch — the measured analogue
of one steady 1F1B period. Stage plans depend only on (stage, layers on the stage), so every
(stage, layers) pair is measured once.

The search restates the native one step for step (initial partition with the OOM shift,
longest stage gives a layer to the shortest stage that lowers the maximum, first improving
move wins, at most L*S rounds); with the simulated oracle it reproduces the native partition
exactly (tests/test_partition_measured.py).
"""
from __future__ import annotations

import json
from fractions import Fraction
from typing import Callable

from . import executor as ex
from . import gpt_profile as gp

Period = Callable[[int, list], Fraction]


def _stage_oom(prof: dict, stage_layers: int, stage: int) -> bool:
    """partition.cpp:100-109 (native `stage_oom`): static share + L_s * n_batch * checkpoint bytes."""
    m, pipe, hw = prof["model"], prof["pipeline"], prof["hardware"]
    nb = min(pipe["n_stages"] - stage, pipe["n_microbatches"])
    ck = next(o for o in m["layer"]["ops"] if o["id"] == m["layer"]["checkpoint_id"])
    share = Fraction(int(m["static_bytes"])) * stage_layers / m["n_layers"]
    return share + stage_layers * nb * int(ck["out_bytes"]) > int(hw["mem_budget_bytes"])


def initial_partition(prof: dict) -> list[int]:
    """partition.cpp:111-142: even split, remainder on later stages, shift toward later stages
    until no stage is OOM."""
    L, S = prof["model"]["n_layers"], prof["pipeline"]["n_stages"]
    if L < S:
        raise ValueError("fewer layers than stages")
    layers = [L // S] * S
    for k in range(L % S):
        layers[S - 1 - k] += 1
    for _ in range(L * S * S):
        bad = next((s for s in range(S) if _stage_oom(prof, layers[s], s)), -1)
        if bad < 0:
            return layers
        if bad == S - 1 or layers[bad] <= 1:
            raise ValueError("no OOM-free initial partition")
        layers[bad] -= 1
        layers[bad + 1] += 1
    raise ValueError("no OOM-free initial partition")


def search_partition(profile_text: str, period: Period) -> dict:
    """Algorithm 1 with `period(stage, layers_per_stage) -> µs` (native greedy_partition)."""
    prof = json.loads(profile_text)
    S = prof["pipeline"]["n_stages"]
    memo: dict[tuple[int, int], Fraction] = {}

    def durations(layers: list[int]) -> list[Fraction]:
        out = []
        for s in range(S):
            key = (s, layers[s])
            if key not in memo:
                memo[key] = Fraction(period(s, list(layers)))
            out.append(memo[key])
        return out

    layers = initial_partition(prof)
    dur = durations(layers)
    moves, iterations = [], 0
    max_iter = prof["model"]["n_layers"] * S
    changed = True
    while changed and iterations < max_iter:
        changed = False
        iterations += 1
        longest = max(range(S), key=lambda s: (dur[s], -s))  # first maximum, as the native loop
        d_long = dur[longest]
        if layers[longest] <= 1:
            break
        order = sorted(range(S), key=lambda s: dur[s])  # stable
        for to in order[:S - 1]:
            if to == longest:
                continue
            cand = list(layers)
            cand[longest] -= 1
            cand[to] += 1
            if any(_stage_oom(prof, cand[s], s) for s in range(S)):
                continue
            cd = durations(cand)
            if max(cd) < d_long:
                layers, dur = cand, cd
                moves.append({"from": longest, "to": to, "accepted": True})
                changed = True
                break
    return {"layers_per_stage": layers, "durations_us": [str(d) for d in dur], "iterations": iterations,
            "moves": moves, "measured": {f"{s}:{n}": float(v) for (s, n), v in sorted(memo.items())}}


def simulated_period(profile_text: str) -> Period:
    """The native planner's steady-period simulation (the reference's stage_period_us)."""
    def period(stage: int, layers: list) -> Fraction:
        return Fraction(ex.plan_for(profile_text, stage, "heu", layers_per_stage=layers)["period_us"])
    return period


def measured_period(c: gp.GPTConfig, profile_text: str, steps: int = 2, warmup: int = 1) -> Period:
    """B200-timed period of one stage: its executor alone on this GPU (TP = 1), iteration time
    over its M microbatches / M, in µs."""
    if c.tp != 1:
        raise ValueError("measured stage periods run at TP = 1 (one GPU)")

    def period(stage: int, layers: list) -> Fraction:
        plan = ex.plan_for(profile_text, stage, "heu", layers_per_stage=layers)
        cfg = ex.make_config(c, layers, exec_opts={"standalone_stage": True})
        e = ex.Executor(profile_text, plan["timeline"], cfg)
        try:
            tok, lab = ex.synthetic_batch(c)
            for _ in range(warmup):
                e.step(tok, lab)
            ms = []
            for _ in range(steps):
                e.step(tok, lab)
                ms.append(e.report()["iteration_ms"])
        finally:
            e.close()
        per_mb_us = 1000.0 * min(ms) / c.n_microbatches
        return Fraction(round(per_mb_us * 1000), 1000)
    return period
