"""Profiler conditions vs the step: the executor-measured operator times of a short standalone stage
(profiler.executor_op_times) under different lengths / warm-ups, against the same operators timed
inside a long stage step — which conditions make the profile B200-true for the simulator.

    python tools/profiler_check.py [--model 7b] [--tp 2]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402
from paper_2406_08756_b200 import profiler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/profiler_check.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base = gp.CONFIGS[a.model]
    c = gp.GPTConfig(**{**base.__dict__, "tp": a.tp, "dropout": 0.1})
    keys = ("qkv", "attn", "mlp_bwd", "attn_bwd", "fc2", "proj", "ln1", "head_fwd", "head_bwd", "embed")
    out = {}
    for name, kw in [("8L_m1", dict(layers=8, micro=1)), ("8L_m2", dict(layers=8, micro=2)),
                     ("8L_m1_w3", dict(layers=8, micro=1, warmup=3, steps=3)), ("4L_m4", dict(layers=4, micro=4))]:
        ms = profiler.executor_op_times(c, **kw)
        out[name] = {k: round(1000 * ms[k], 1) for k in keys if k in ms}
        print(name, json.dumps(out[name]), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
