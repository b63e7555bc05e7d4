"""One TP rank of a TP·PP stage on one B200, with the plan's comm windows (exec.comm_standin_us).

The headline configuration (GPT-7B, micro-batch 32, TP2·PP4, 8 microbatches) needs eight GPUs.
Each stage's TP-rank-0 executor runs alone (exec.standalone_stage: pipeline receives read synthetic
activations / gradients, sends are skipped) with every TP all-reduce replaced by a stand-in kernel
that holds the TP stream for the transfer time the plan's window capacities assume
(2(t-1)/t * [T,h] bf16 / profiler.NVLINK_BUS_GBS). The recompute items the plan files into those
windows (expand_plan_to_stage, heusched.cpp:372-405) run on the side stream against it, so window
overlap, on-demand recompute and waits are measured on real B200 kernels. The SM and HBM traffic of
a real NCCL all-reduce is not modelled (the stand-in sleeps on `ctas` CTAs).

Pipeline bubbles: alone, a stage's receives complete at once, so the cool-down stall-fill items
(expand_plan_to_stage, heusched.cpp:374-380), planned into the wait for the next gradient, would
meet no wait. With `bubbles`, the stall the native simulator predicts before each backward's
gradient receive on this stage (its trace, pipesim.cpp:620-646) is held by a stand-in kernel on
the gradient stream (exec.standin_grad_wait_us), so the stage runs its pipelined timeline: the
stall-fill recomputes overlap it, and the iteration includes the stage's warm-up / cool-down
bubbles. Forward (activation) receive stalls are not emulated.
"""
from __future__ import annotations

import json
from fractions import Fraction

from . import executor as ex
from . import gpt_profile as gp
from . import planner
from . import profiler


def standin_us(c: gp.GPTConfig) -> float:
    """Modelled TP all-reduce time of one [T, h] bf16 tensor (the profiler's comm model)."""
    return 2.0 * (c.tp - 1) / c.tp * (2 * c.tokens * c.hidden) / (profiler.NVLINK_BUS_GBS * 1e3)


def simulated_grad_waits(text: str, stage: int, n_micro: int) -> list[float]:
    """Per microbatch m: the stall (µs) the simulator puts on `stage` before B(m) starts (its
    gradient receive), from the native simulator's CSV trace of the HEU plans."""
    rows = [r.split(",") for r in planner.simulate_text(text, "heu", fmt="csv").splitlines()[1:]]
    waits, pending = [0.0] * n_micro, 0.0
    for r in rows:
        if r[0] != str(stage):
            continue
        kind = r[2]
        if kind == "stall":
            pending += float(r[5]) - float(r[4])
        elif kind in ("p2p", "stall_recompute", "recompute"):
            continue
        elif kind in ("bwd", "comm_bwd"):
            waits[int(r[1])] += pending
            pending = 0.0
        else:  # a forward receive stall: not emulated
            pending = 0.0
    return waits


def simulated_stage_ms(text: str, stage: int) -> float:
    """The simulator's prediction of what the emulation measures for `stage` (ms): the stage's span in
    the native simulator's HEU trace (first to last event) minus the stalls before forward passes
    (activation receives, which the emulation does not hold)."""
    rows = [r.split(",") for r in planner.simulate_text(text, "heu", fmt="csv").splitlines()[1:]]
    mine = [r for r in rows if r[0] == str(stage) and r[2] != "p2p"]
    if not mine:
        return 0.0
    start = min(float(r[4]) for r in mine)
    end = max(float(r[5]) for r in mine)
    fwd_stall, pending = 0.0, 0.0
    for r in mine:
        if r[2] == "stall":
            pending += float(r[5]) - float(r[4])
        elif r[2] in ("fwd", "comm_fwd"):
            fwd_stall += pending
            pending = 0.0
        elif r[2] in ("bwd", "comm_bwd"):
            pending = 0.0
    return (end - start - fwd_stall) / 1000.0


def run_stage(text: str, timeline: dict, c: gp.GPTConfig, layers, opts: dict, tok, lab, steps: int = 2,
              warmup: int = 1) -> dict:
    """The stage's executor alone: best of `steps` iterations after `warmup`."""
    import torch
    cfg = ex.make_config(c, layers, exec_opts={"standalone_stage": True, **opts})
    from .clocks import ClockSampler
    e = ex.Executor(text, timeline, cfg)
    try:
        for _ in range(warmup):
            e.step(tok, lab)
        reps = []
        sampler = ClockSampler(0)
        with sampler:
            for _ in range(steps):
                e.step(tok, lab)
                reps.append(e.report())
        clk = sampler.summary()
    finally:
        e.close()
        torch.cuda.empty_cache()
    r = min(reps, key=lambda x: x["iteration_ms"])
    import statistics
    op_ms = {k: round(statistics.median(v), 4) for k, v in r.get("op_timing_ms", {}).items()}
    keys = ("iteration_ms", "comm_ms", "busy_ms", "recv_wait_ms", "exposed_recompute_ms", "recompute_on_demand_ms",
            "recompute_overlapped_ms", "wait_on_recompute_ms", "recompute_launches", "pool_high_water_bytes",
            "elide_fill_ms")
    out = {k: r[k] for k in keys if k in r} | {"iteration_ms_each": [round(x["iteration_ms"], 3) for x in reps],
                                               "sm_mhz_median": clk.get("sm_mhz")}
    if op_ms:
        out["op_timing_median_ms"] = op_ms
    return out


def emulate(c: gp.GPTConfig, text: str, stages, *, steps: int = 2, warmup: int = 1, ctas: int = 16,
            variants=("heu", "elided", "full_recompute"), bubbles: bool = True, op_timing: bool = False,
            extra_opts: dict | None = None) -> dict:
    """Per stage: its HEU plan, the same plan with recompute elided (no-recompute floor), Megatron full
    recompute and (variant "selective") Megatron selective recompute, each as one TP rank with stand-in
    all-reduces."""
    std = {"comm_standin_us": standin_us(c), "comm_standin_ctas": ctas, **(extra_opts or {})}
    tok, lab = ex.synthetic_batch(c)
    out = {}
    for s in stages:
        waits = simulated_grad_waits(text, s, c.n_microbatches) if bubbles else []
        std = {**std, "standin_grad_wait_us": waits}
        heu = ex.plan_for(text, s, "heu")
        layers = heu["layers_per_stage"]
        pj = json.loads(heu["plan_json"])
        row = {"layers_per_stage": layers, "plan": {k: pj[k] for k in ("S", "phase_assignment", "peak_bytes")},
               "simulated_period_us": heu["period_us"],
               "simulated_stage_ms": round(simulated_stage_ms(text, s), 3),
               "grad_wait_us": [round(w, 1) for w in waits]}
        for v in variants:
            try:
                if v == "heu":
                    row[v] = run_stage(text, heu["timeline"], c, layers, {**std, "op_timing": op_timing}, tok, lab,
                                       steps, warmup)
                elif v == "elided":  # stand-in buffers filled with noise (realistic operands), fill time excluded
                    row[v] = run_stage(text, heu["timeline"], c, layers,
                                       {**std, "elide_recompute": True, "elide_fill": True}, tok, lab, steps, warmup)
                    row[v]["iteration_ms"] -= row[v].get("elide_fill_ms", 0.0)
                else:  # Megatron baselines: "full_recompute" (keep the checkpoint only), "selective" (core attention)
                    base = ex.plan_for(text, s, "full" if v == "full_recompute" else v)
                    row[v] = run_stage(text, base["timeline"], c, layers, std, tok, lab, steps, warmup)
                    peak = json.loads(base["plan_json"])["peak_bytes"]
                    row[v]["plan_peak_bytes"] = peak
                    row[v]["fits_budget"] = int(peak) <= json.loads(text)["hardware"]["mem_budget_bytes"]
            except ex.LynxError as err:
                row[v] = {"error": str(err)[:200]}
        # contention: the window / stall-fill regenerations' measured side-stream time (beside a 16-CTA
        # all-reduce stand-in) against their cost in the profile (measured alone)
        prof = json.loads(text)["model"]["layer"]["ops"]
        cost_us = {i: float(Fraction(str(o["time_us"]))) for i, o in enumerate(prof)}
        side_cost = sum(cost_us[it["op"]] for it in heu["timeline"]["items"] if it["host"] in ("window", "stall"))
        row["side_items_profile_ms"] = round(side_cost / 1000.0, 3)
        hr = row.get("heu", {})
        if "iteration_ms" in hr and side_cost > 0:
            row["side_items_measured_over_profile"] = round(hr["recompute_overlapped_ms"] / (side_cost / 1000.0), 4)
        if "iteration_ms" in hr:
            row["exposed_fraction_of_iteration"] = round(hr["exposed_recompute_ms"] / hr["iteration_ms"], 4)
            rc = hr["recompute_on_demand_ms"] + hr["recompute_overlapped_ms"]
            row["exposed_fraction_of_recompute"] = round(hr["exposed_recompute_ms"] / rc, 4) if rc else 0.0
            if row["simulated_stage_ms"]:  # simulator fidelity: predicted / measured stage time
                row["simulated_over_measured"] = round(row["simulated_stage_ms"] / hr["iteration_ms"], 4)
            if "iteration_ms" in row.get("elided", {}):
                row["crosscheck_ms"] = round(hr["iteration_ms"] - row["elided"]["iteration_ms"], 3)
        out[str(s)] = row
    return out
