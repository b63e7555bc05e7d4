"""Compare a plan's step time with the recompute-elided timing mode on a small GPT-7B slice.

    python tools/elide_check.py [layers] [micro_batch]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import executor as ex  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    mb = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    c = gp.GPTConfig(**{**gp.CONFIGS["7b"].__dict__, "n_layers": L, "micro_batch": mb, "dropout": 0.1,
                                  "tp": 1, "pp": 1, "n_microbatches": 1})
    static = gp.BYTES_PER_PARAM_STATIC * c.params()
    c.mem_budget_bytes = static + 6 * 2**30 * L // 4
    text = gp.profile_text(c)
    plan = ex.plan_for(text, 0, "heu")
    print("plan", json.loads(plan["plan_json"])["S"], "items", len(plan["timeline"]["items"]), flush=True)
    tok, lab = ex.synthetic_batch(c)
    for opts in ({}, {"elide_recompute": True}, {}, {"elide_recompute": True}):
        e = ex.Executor(text, plan["timeline"], ex.make_config(c, [L], exec_opts=opts))
        ms = []
        for _ in range(4):
            e.step(tok, lab)
            ms.append(round(e.report()["iteration_ms"], 2))
        r = e.report()
        print(opts, ms, "busy", round(r["busy_ms"], 1), "exposed", round(r["exposed_recompute_ms"], 1),
              "launches", r["kernel_launches"], "loss", r["loss"], flush=True)
        e.close()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
