"""OPT plans at GPT scale through an external MILP solver.

The reference's OPT model (paper Eqs. 1-10; proj/src/optsched.cpp:54-214) places every
recompute of one stage's unrolled 1F1B operator sequence on a phase grid: Θ(n²) booleans, with
n = M x (layer ops) x L_s. Its embedded branch-and-bound (optsched.cpp:216-243) is exact but
only finishes on small graphs; a 7B stage has ~10^6 variables.

This module takes the OPT program over a *slice* of `slice_layers` consecutive layers (the
slice's static share plus the stage's activation budget minus a reserve for the other layers'
retained tensors, see include/lynx_rt.h: lynx_plan_opt_export), solves it with HiGHS
(`scipy.optimize.milp`), and hands the 0/1 answer back to the native planner, which
  1. checks it *exactly* in rational arithmetic (check_schedule, optsched.cpp:245-338) —
     HiGHS works in doubles, so a schedule that is infeasible by a few bytes is rejected and the
     slice is re-solved with a slightly smaller budget;
  3. (plan_stage) bisects the reserve until the replicated timeline fits the stage budget under
     the native simulator's ledger.
  2. converts it with timeline_from_opt_schedule (report_io.cpp:187-294) and replicates the
     slice over the stage's layers.
The resulting timeline is an ordinary StageRecomputeTimeline: the native simulator scores it
(`simulate_timelines_text`, ledger included) and the GPU executor replays it like a HEU plan.

The solver is the only thing that differs from the reference's OPT path; everything it
produces passes through the same exact checker.
"""
from __future__ import annotations

import time
from fractions import Fraction

import numpy as np

from . import planner


def _milp(model: dict, time_limit_s: float):
    from scipy.optimize import Bounds, LinearConstraint, milp
    from scipy.sparse import coo_matrix

    n, m = model["n_vars"], model["n_rows"]
    c = np.zeros(n)
    for v, k in model["objective"]:
        c[v] += k
    row = np.asarray(model["row"], dtype=np.int64)
    col = np.asarray(model["col"], dtype=np.int64)
    val = np.asarray(model["val"], dtype=np.float64)
    rhs = np.asarray(model["rhs"], dtype=np.float64)
    sense = np.asarray(model["sense"], dtype=np.int64)
    lo, hi = np.asarray(model["lo"], dtype=np.float64), np.asarray(model["hi"], dtype=np.float64)
    integ = np.asarray(model["integer"], dtype=np.int64)
    # the continuous ledger variables are byte counts: solve them in units of the largest
    # coefficient (the largest tensor; column scaling), then scale every row by its largest
    # coefficient. Unscaled, a 7B ledger row has a 1 next to 1e9-byte coefficients and HiGHS
    # drops the 1 as a sub-tolerance matrix entry.
    unit = float(np.max(np.abs(val))) if len(val) else 1.0
    colscale = np.where(integ == 0, max(unit, 1.0), 1.0)
    val = val * colscale[col]
    lo, hi = lo / colscale, hi / colscale
    c = c * colscale
    scale = np.ones(m)
    if len(val):
        np.maximum.at(scale, row, np.abs(val))
    val = val / scale[row]
    rhs = rhs / scale
    A = coo_matrix((val, (row, col)), shape=(m, n)).tocsr()
    lb = np.where(sense >= 0, rhs, -np.inf)
    ub = np.where(sense <= 0, rhs, np.inf)
    res = milp(c, constraints=LinearConstraint(A, lb, ub), integrality=integ, bounds=Bounds(lo, hi),
               options={"time_limit": float(time_limit_s), "mip_rel_gap": 0.0, "disp": False})
    return res


def _pairs(x, grid, strict: bool):
    out = []
    for t, vars_t in enumerate(grid):
        for i, v in enumerate(vars_t):
            if strict and i >= t:
                continue
            if x[v] > 0.5:
                out.append([t, i])
    return out


def solve_stage(profile_text: str, stage: int, layers_per_stage=None, slice_layers: int = 1,
                time_limit_s: float = 60.0, max_tries: int = 4, reserve_bytes: int | None = None) -> dict:
    """OPT timeline for one stage from a HiGHS-solved layer slice.

    Returns {timeline, cost_us (slice, exact), status, slice_layers, n_vars, n_rows, solve_s,
    reserve_bytes, tries}. Raises RuntimeError when no exactly-feasible schedule was found."""
    reserve = reserve_bytes
    tries = []
    for _ in range(max_tries):
        rs = None if reserve is None else str(int(reserve))
        model = planner.opt_export_text(profile_text, stage, layers_per_stage, slice_layers, rs)
        t0 = time.perf_counter()
        res = _milp(model, time_limit_s)
        dt = time.perf_counter() - t0
        if res.x is None:
            raise RuntimeError(f"HiGHS found no schedule for stage {stage} ({res.message})")
        status = "optimal" if res.status == 0 else "feasible"
        sched = {"status": status, "keep": _pairs(res.x, model["S"], False),
                 "recompute": _pairs(res.x, model["R"], True)}
        out, st = planner.opt_timeline_text(profile_text, stage, sched, layers_per_stage, slice_layers, rs)
        tries.append({"reserve_bytes": rs, "status": status, "solve_s": round(dt, 3),
                      "objective": float(res.fun), "issues": out["issues"][:300]})
        if st == 0:
            return {"timeline": out["timeline"], "cost_us": out["cost_us"], "status": status,
                    "slice_layers": model["slice_layers"], "stage_layers": model["stage_layers"],
                    "n_ops": model["n_ops"], "n_vars": model["n_vars"], "n_rows": model["n_rows"],
                    "n_recompute": out["n_recompute"], "n_overlapped": out["n_overlapped"],
                    "completed_owners": out.get("completed_owners", 0),
                    "solve_s": round(dt, 3), "reserve_bytes": rs, "slice_budget_bytes": model["budget_bytes"],
                    "tries": tries}
        # round-off in the byte rows: retry just inside the budget
        act = int(Fraction(model["stage_activation_bytes"]))
        base = int(reserve) if reserve is not None else act - (model["budget_bytes"] - model["static_bytes"])
        reserve = base + max(act // 1000, 1)
    raise RuntimeError(f"no exactly-feasible OPT schedule for stage {stage}: {tries[-1]['issues']}")


def _stage_peak(profile_text: str, layers_per_stage, stage: int, timeline: dict, others: list) -> int:
    tls = list(others)
    tls[stage] = timeline
    sim = planner.simulate_timelines_text(profile_text, layers_per_stage, tls)
    return int(Fraction(sim["memory_peaks"][stage]))


def plan_stage(profile_text: str, stage: int, layers_per_stage, slice_layers: int = 1, time_limit_s: float = 60.0,
               search_steps: int = 8, others=None) -> dict:
    """The smallest reserve whose replicated slice timeline fits the stage's real budget.

    A slice is solved with the stage's activation budget minus `reserve` bytes, the room the
    replicated copies' retained tensors need. Reserve 0 lets the slice retain as if it were alone
    (the replicated stage then overflows); reserve = all of it leaves the slice nothing. Each
    candidate timeline is scored by the native simulator's ledger over the whole stage
    (`memory_peaks`, the reference's pipesim.cpp:722-736 rules): overflow -> more reserve, an
    infeasible slice -> less, bisected `search_steps` times."""
    import json
    budget = int(json.loads(profile_text)["hardware"]["mem_budget_bytes"])
    if others is None:
        others = [planner.stage_plan_text(profile_text, s, layers_per_stage)["timeline"]
                  for s in range(len(layers_per_stage))]
    act = int(Fraction(planner.opt_export_text(profile_text, stage, layers_per_stage, slice_layers)
                       ["stage_activation_bytes"]))
    evaluated = []

    def attempt(reserve: int):
        try:
            r = solve_stage(profile_text, stage, layers_per_stage, slice_layers, time_limit_s, max_tries=2,
                            reserve_bytes=reserve)
        except RuntimeError as err:
            evaluated.append({"reserve_bytes": reserve, "error": str(err)[:120]})
            return None, "infeasible"
        peak = _stage_peak(profile_text, layers_per_stage, stage, r["timeline"], others)
        r["stage_peak_bytes"] = peak
        evaluated.append({"reserve_bytes": reserve, "peak": peak, "cost_us": r["cost_us"], "fits": peak <= budget})
        return (r, "ok") if peak <= budget else (None, "over")

    best, kind = attempt(0)
    lo, hi = 0, act  # invariant: reserve lo overflows (or is the answer), reserve hi is infeasible or fits
    if best is None and layers_per_stage[stage] != slice_layers:
        for _ in range(search_steps):
            mid = (lo + hi) // 2
            r, kind = attempt(mid)
            if r is not None:
                best, hi = r, mid  # fits: try to give the slice more
            elif kind == "over":
                lo = mid
            else:
                hi = mid
    if best is None:
        raise RuntimeError(f"no reserve gives a timeline that fits stage {stage}: {evaluated}")
    best["search"] = evaluated
    return best


def plan_all(profile_text: str, layers_per_stage, slice_layers: int = 1, time_limit_s: float = 60.0,
             search_steps: int = 8) -> dict:
    """OPT timelines for every stage plus the native simulator's report of the whole pipeline."""
    heu = [planner.stage_plan_text(profile_text, s, layers_per_stage)["timeline"]
           for s in range(len(layers_per_stage))]
    stages = [plan_stage(profile_text, s, layers_per_stage, slice_layers, time_limit_s, search_steps, heu)
              for s in range(len(layers_per_stage))]
    sim = planner.simulate_timelines_text(profile_text, layers_per_stage, [x["timeline"] for x in stages])
    return {"stages": stages, "iteration_us": sim["iteration_us_exact"], "memory_peaks": sim["memory_peaks"],
            "report": sim["report"]}
