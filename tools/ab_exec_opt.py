"""A/B of one executor option on the bench workload (GPT-7B, N = 1, HEU plan from B200-measured op
times): two executors in turn, the same plan and batch, alternating steps, step times from the
executor's own CUDA events.

    python tools/ab_exec_opt.py dw_concurrent [--steps 6]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("option")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--margin", type=float, default=8.0)
    args = ap.parse_args()
    import numpy as np
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
    tok, lab = ex.synthetic_batch(c)
    res = {True: [], False: []}
    losses = {}
    for i in range(args.steps):
        for val in (True, False) if i % 2 == 0 else (False, True):
            e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"],
                                                                  exec_opts={args.option: val}))
            e.step(tok, lab)  # warm-up
            loss = e.step(tok, lab)
            res[val].append(e.report()["iteration_ms"])
            losses.setdefault(val, loss)
            e.close()
            torch.cuda.empty_cache()
    out = {str(k): {"median_ms": float(np.median(v)), "all_ms": [round(x, 1) for x in v]} for k, v in res.items()}
    out["same_loss"] = losses[True] == losses[False]
    print(json.dumps({args.option: out}))


if __name__ == "__main__":
    main()
