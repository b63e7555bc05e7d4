"""Host issue cost of a training step: host time to enqueue the step vs device time of the step.

For configurations whose kernels are short (the tiny parity config, small pipeline stages) the
step can become bound by the host issuing launches; this prints, per configuration, the device
iteration time, the host time spent issuing (before the final synchronisation) and the number of
kernels, with and without CUDA-graph replay of the step (exec.graph).

    python tools/host_issue.py [--graph]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_08756_b200 import executor as ex  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402


def measure(c, plan_kind, opts, steps=6):
    text = gp.profile_text(c)
    plan = ex.plan_for(text, 0, plan_kind)
    e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"], exec_opts=opts))
    tok, lab = ex.synthetic_batch(c)
    try:
        for _ in range(2):
            e.step(tok, lab)
        reps = []
        for _ in range(steps):
            e.step(tok, lab)
            reps.append(e.report())
    finally:
        e.close()
    r = sorted(reps, key=lambda x: x["iteration_ms"])[len(reps) // 2]
    toks = c.tokens * c.n_microbatches
    return {"iteration_ms": round(r["iteration_ms"], 3), "host_issue_ms": round(r["host_issue_ms"], 3),
            "kernel_launches": r["kernel_launches"], "tokens_per_s": round(toks / (r["iteration_ms"] / 1e3), 1),
            "host_us_per_launch": round(1e3 * r["host_issue_ms"] / max(1, r["kernel_launches"]), 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--out", default="gpurun_out/host_issue.json")
    a = ap.parse_args()
    cfgs = {
        "tiny (BASELINE configs[0]) M=8": (gp.GPTConfig("gpt-tiny", 4, 512, 8, 256, 2, 50304, 1, 1, 8, dropout=0.1), "heu"),
        "tiny M=8 full recompute": (gp.GPTConfig("gpt-tiny", 4, 512, 8, 256, 2, 50304, 1, 1, 8, dropout=0.1), "full"),
    }
    out = {}
    for name, (c, kind) in cfgs.items():
        out[name] = {"eager": measure(c, kind, {})}
        if a.graph:
            out[name]["graph"] = measure(c, kind, {"graph": True})
        print(name, json.dumps(out[name]), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
