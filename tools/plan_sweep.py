"""Per-step iteration times of the executor under different recompute plans (fresh executor each).

    python tools/plan_sweep.py [--model 7b] [--plans full,heu,full,heu] [--steps 4] [--trace out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2406_08756_b200 import executor as ex  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--plans", default="full,heu,full,heu")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--micro-batch", type=int, default=0)
    ap.add_argument("--trace", default="")
    a = ap.parse_args()
    args = argparse.Namespace(model=a.model, microbatches=0, micro_batch=a.micro_batch, plan="heu")
    c = bench.config_for(1, args)
    if a.layers:
        c.n_layers = a.layers
    _, total = torch.cuda.mem_get_info()
    c.mem_budget_bytes = bench.device_budget(c, total)
    text = gp.profile_text(c)
    tok, lab = ex.synthetic_batch(c)
    for plan in a.plans.split(","):
        p = ex.plan_for(text, 0, plan)
        cfg = ex.make_config(c, p["layers_per_stage"], exec_opts={"trace": bool(a.trace)})
        e = ex.Executor(text, p["timeline"], cfg)
        rows = []
        for _ in range(a.steps):
            e.step(tok, lab)
            r = e.report()
            rows.append({k: round(r[k], 2) for k in ("iteration_ms", "busy_ms", "recompute_on_demand_ms")})
        print(json.dumps({"plan": plan, "S": json.loads(p["plan_json"])["S"], "steps": rows,
                          "pool_hw_gb": round(r["pool_high_water_bytes"] / 1e9, 1)}), flush=True)
        if a.trace:
            with open(a.trace.replace(".json", f"_{plan}.json"), "w") as f:
                f.write(e.trace("chrome"))
        e.close()


if __name__ == "__main__":
    main()
