"""In-step time per operator (exec option probe_ops: one CUDA event after every operator launch on
its stream; consecutive differences = the operator's kernels plus any idle gap before them).

    python tools/step_ops.py [--steps 4] [--margin 8] [--out gpurun_out/step_ops.json]

Same workload and plan as `bench.py` at N = 1 (GPT-7B, B200-measured operator times, HEU).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--margin", type=float, default=8.0)
    ap.add_argument("--out", default="gpurun_out/step_ops.json")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    from paper_2406_08756_b200 import profiler

    class A:
        model, microbatches, micro_batch = "7b", None, None

    c = bench.config_for(1, A)
    total = torch.cuda.mem_get_info()[1]
    c.mem_budget_bytes = bench.device_budget(c, total, args.margin)
    times = profiler.measure_op_times(c)
    torch.cuda.empty_cache()
    text = gp.profile_text(c, times=times)
    plan = ex.plan_for(text, 0)
    e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"],
                                                          exec_opts={"probe_ops": True}))
    tok, lab = ex.synthetic_batch(c)
    reps, clocks = [], []
    cs = bench.ClockSampler(0)  # NVML initialised once, before the steps (as in bench.py)
    for _ in range(args.steps):
        cs.rows.clear()
        cs._stop.clear()
        with cs:
            e.step(tok, lab)
        clocks.append(cs.summary())
        reps.append(e.report())
    e.close()
    r = reps[-1]
    ops = sorted(r["probe_ops"].items(), key=lambda kv: -kv[1][1])
    print("steps", [round(x["iteration_ms"], 1) for x in reps], "clocks", [c_["sm_mhz"] for c_ in clocks])
    for x in reps:
        print(f"  step {x['step']}: {x['iteration_ms']:.1f} ms, host issue {x['host_issue_ms']:.1f} ms, "
              f"alloc host {x['alloc_host_ms']:.1f} ms (max {x['alloc_host_max_ms']:.1f}), "
              f"pool reserved {x['pool_reserved_bytes'] / 1e9:.2f} GB, high {x['pool_high_water_bytes'] / 1e9:.2f} GB")
    print(f"iteration {r['iteration_ms']:.1f} ms; main-stream op sum {r['probe_ops_main_ms']:.1f} ms; "
          f"side {r['probe_ops_side_ms']:.1f} ms; plan {json.loads(plan['plan_json'])['S']}")
    for k, (n, ms) in ops:
        print(f"  {ms:9.2f} ms {n:5d}  {k}")
    with open(args.out, "w") as f:
        json.dump({"iteration_ms": [x["iteration_ms"] for x in reps], "clocks": clocks, "last": r}, f, indent=1)


if __name__ == "__main__":
    main()
