"""HEU vs OPT-at-scale (HiGHS on a layer slice, opt_milp.py) on the GPT pipeline profiles.

For each config: the native partition, HEU timelines (the reference's planner) and OPT-slice
timelines for every stage, each scored by the native simulator (iteration time, ledger peaks).
Writes one JSON document (default profiles/r01_opt_vs_heu.json).

    python tools/opt_vs_heu.py [--configs 1.3b 7b] [--slice 1] [--out profiles/r01_opt_vs_heu.json]
"""
import argparse
import json
import os
import sys
import time
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402
from paper_2406_08756_b200 import opt_milp, planner  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["1.3b", "7b"])
    ap.add_argument("--slice", type=int, default=1)
    ap.add_argument("--time-limit", type=float, default=120.0)
    ap.add_argument("--budget-gb", type=float, nargs="*", default=[0.0],
                    help="mem_budget_bytes overrides in GB (0 = the config's own)")
    ap.add_argument("--out", default="profiles/r01_opt_vs_heu.json")
    args = ap.parse_args()
    out = {"note": "estimated operator times (gpt_profile.estimate_times), TPxPP of CONFIGS; "
                   "iteration_us from the native simulator (the reference's simulate())", "configs": {}}
    for name, budget_gb in [(n, b) for n in args.configs for b in args.budget_gb]:
        c = gp.GPTConfig(**gp.CONFIGS[name].__dict__)
        if budget_gb:
            c.mem_budget_bytes = int(budget_gb * 1e9)
            name = f"{name}@{budget_gb:g}GB"
        text = gp.profile_text(c)
        part = json.loads(planner.partition_text(text))["layers_per_stage"]
        t0 = time.perf_counter()
        heu = [planner.stage_plan_text(text, s, part) for s in range(len(part))]
        t_heu = time.perf_counter() - t0
        sim_h = planner.simulate_timelines_text(text, part, [h["timeline"] for h in heu])
        t0 = time.perf_counter()
        opt = opt_milp.plan_all(text, part, args.slice, args.time_limit)
        t_opt = time.perf_counter() - t0
        rep_h, rep_o = sim_h["report"], opt["report"]
        out["configs"][name] = {
            "tp": c.tp, "pp": c.pp, "n_microbatches": c.n_microbatches, "layers_per_stage": part,
            "budget_bytes": json.loads(text)["hardware"]["mem_budget_bytes"],
            "heu": {"iteration_us": float(Fraction(sim_h["iteration_us_exact"])),
                    "memory_peaks": [int(Fraction(p)) for p in sim_h["memory_peaks"]],
                    "items": [len(h["timeline"]["items"]) for h in heu], "plan_s": round(t_heu, 3),
                    "recompute_on_demand_us": [s.get("recompute_on_demand_us") for s in rep_h.get("stages", [])]},
            "opt_slice": {"iteration_us": float(Fraction(opt["iteration_us"])),
                          "memory_peaks": [int(Fraction(p)) for p in opt["memory_peaks"]],
                          "items": [len(s["timeline"]["items"]) for s in opt["stages"]],
                          "overlapped": [s["n_overlapped"] for s in opt["stages"]],
                          "completed_owners": [s["completed_owners"] for s in opt["stages"]],
                          "slice_ops": [s["n_ops"] for s in opt["stages"]],
                          "vars": [s["n_vars"] for s in opt["stages"]],
                          "solve_s": [s["solve_s"] for s in opt["stages"]], "plan_s": round(t_opt, 3),
                          "recompute_on_demand_us": [s.get("recompute_on_demand_us")
                                                     for s in rep_o.get("stages", [])]},
        }
        print(name, json.dumps(out["configs"][name]), flush=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
