"""Where recompute time goes: the span metric vs T(plan) - T(elided), operator by operator (B200).

The executor reports exposed recompute two ways: the span metric (on-demand recompute
kernels on the main stream + main-stream waits on side-stream regenerations) and the cross-check
T(plan) - T(same plan, recompute launches elided). This runs the bench's workload (GPT-7B, TP1,
micro-batch 32, HEU plan from B200-measured operator times) as
  plan          the HEU plan as the bench runs it
  elided        recompute launches skipped, consumers read stale pool memory
  elided_fill   the same, each stand-in buffer first filled with bf16 noise (fill time reported and
                subtracted), so consumers read realistic operands
and, per variant, the SM clock under load (NVML) and the in-step time of every operator
(exec.probe_ops; regenerations tagged "re: "), so the difference between the measures can be
attributed: recompute kernels themselves, and the change in the other operators' time.

    python tools/recompute_accounting.py [--model 7b] [--out gpurun_out/recompute_accounting.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_08756_b200 import executor as ex  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402
from paper_2406_08756_b200 import profiler  # noqa: E402


def run(text, timeline, cfg_fn, tok, lab, opts, steps, warmup):
    e = ex.Executor(text, timeline, cfg_fn({**opts}))
    try:
        for _ in range(warmup):
            e.step(tok, lab)
        sampler = bench.ClockSampler(0)
        reps = []
        with sampler as clk:
            for _ in range(steps):
                e.step(tok, lab)
                reps.append(e.report())
        r = sorted(reps, key=lambda x: x["iteration_ms"])[len(reps) // 2]
        return r, clk.summary(), [round(x["iteration_ms"], 2) for x in reps]
    finally:
        e.close()
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--pool-internal-deps", action="store_true")
    ap.add_argument("--out", default="gpurun_out/recompute_accounting.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base = gp.CONFIGS[a.model]
    c = gp.GPTConfig(**{**base.__dict__, "tp": 1, "pp": 1, "n_microbatches": 1, "dropout": 0.1})
    times = profiler.measure_op_times(c)
    torch.cuda.empty_cache()
    _, total = torch.cuda.mem_get_info()
    c.mem_budget_bytes = bench.device_budget(c, total)
    text = gp.profile_text(c, times=times)
    plan = ex.plan_for(text, 0, "heu")
    tok, lab = ex.synthetic_batch(c)
    lps = plan["layers_per_stage"]

    def cfg(opts):
        return ex.make_config(c, lps, exec_opts={"pool_internal_deps": a.pool_internal_deps, **opts})

    out = {"workload": f"gpt-{a.model} TP1 micro-batch {c.micro_batch}, HEU plan {json.loads(plan['plan_json'])['S']}",
           "variants": {}}
    variants = {"plan": {}, "elided": {"elide_recompute": True},
                "elided_fill": {"elide_recompute": True, "elide_fill": True}}
    for name, opts in variants.items():
        r, clk, each = run(text, plan["timeline"], cfg, tok, lab, opts, a.steps, a.warmup)
        rp, _, _ = run(text, plan["timeline"], cfg, tok, lab, {**opts, "probe_ops": True}, 2, 1)
        out["variants"][name] = {"iteration_ms": r["iteration_ms"], "exposed_recompute_ms": r["exposed_recompute_ms"],
                                 "recompute_on_demand_ms": r["recompute_on_demand_ms"],
                                 "elide_fill_ms": r.get("elide_fill_ms", 0.0), "clocks": clk, "steps_ms": each,
                                 "probe_ops": rp.get("probe_ops", {}), "probe_main_ms": rp.get("probe_ops_main_ms")}
        print(name, json.dumps({k: v for k, v in out["variants"][name].items() if k != "probe_ops"}), flush=True)
    v = out["variants"]
    p_ops = {k: x[1] for k, x in v["plan"]["probe_ops"].items()}
    for ref in ("elided", "elided_fill"):
        e_ops = {k: x[1] for k, x in v[ref]["probe_ops"].items()}
        shared = sorted(set(p_ops) & set(e_ops), key=lambda k: -(p_ops[k] - e_ops[k]))
        recompute_ms = sum(x for k, x in p_ops.items() if k.startswith("re: "))
        out[f"plan_minus_{ref}"] = {
            "iteration_ms": round(v["plan"]["iteration_ms"] - (v[ref]["iteration_ms"] - v[ref]["elide_fill_ms"]), 3),
            "span_metric_ms": round(v["plan"]["exposed_recompute_ms"], 3),
            "recompute_ops_ms (probe)": round(recompute_ms, 3),
            "other_ops_delta_ms (probe)": round(sum(p_ops[k] - e_ops[k] for k in shared if not k.startswith("re: ")), 3),
            "largest_other_op_deltas_ms": {k: round(p_ops[k] - e_ops[k], 3) for k in shared[:12]
                                           if not k.startswith("re: ")}}
        print(ref, json.dumps(out[f"plan_minus_{ref}"]), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
