"""Per-element CUDA-event trace of one emulated TP·PP stage (stand-in all-reduces), for finding
where the main stream waits on window recomputes.

    python tools/trace_stage.py [--model 7b] [--stage 0] [--out gpurun_out/trace_stage0.csv]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_08756_b200 import executor as ex  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402
from paper_2406_08756_b200 import profiler  # noqa: E402
from paper_2406_08756_b200 import stage_emulation as se  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--stage", type=int, default=0)
    ap.add_argument("--budget-gb", type=float, default=0.0)
    ap.add_argument("--out", default="gpurun_out/trace_stage0.csv")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    c = gp.GPTConfig(**{**gp.CONFIGS[a.model].__dict__, "dropout": 0.1})
    times = profiler.measure_op_times(c)
    torch.cuda.empty_cache()
    _, total = torch.cuda.mem_get_info()
    c.mem_budget_bytes = int(a.budget_gb * 1e9) if a.budget_gb else bench.device_budget(c, total)
    text = gp.profile_text(c, times=times)
    plan = ex.plan_for(text, a.stage, "heu")
    opts = {"standalone_stage": True, "trace": True, "comm_standin_us": se.standin_us(c)}
    e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"], exec_opts=opts))
    tok, lab = ex.synthetic_batch(c)
    e.step(tok, lab)
    e.step(tok, lab)
    rep = e.report()
    with open(a.out, "w") as f:
        f.write(e.trace("csv"))
    with open(a.out.replace(".csv", ".timeline.json"), "w") as f:
        import json
        json.dump(plan["timeline"], f)
    e.close()
    print({k: rep[k] for k in ("iteration_ms", "exposed_recompute_ms", "wait_on_recompute_ms",
                               "recompute_overlapped_ms")})


if __name__ == "__main__":
    main()
