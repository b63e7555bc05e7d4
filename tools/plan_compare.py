"""Run the GPT-7B N=1 executor under two HEU memory margins and print per-step times.

    python tools/plan_compare.py 12 7
"""
import json
import sys
import time
from fractions import Fraction

import torch

sys.path.insert(0, ".")
import importlib.util  # noqa: E402

from paper_2406_08756_b200 import executor as ex  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402

spec = importlib.util.spec_from_file_location("bench", "bench.py")
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def main():
    margins = [float(x) for x in sys.argv[1:]] or [12.0]
    prof = json.load(open("profiles/r01_bench_n1.json"))
    times = {k: Fraction(v).limit_denominator(1000) for k, v in prof["recompute"]["op_times_us"].items()}

    class A:
        model, micro_batch, microbatches = "7b", 0, 0

    c = bench.config_for(1, A())
    for m in margins:
        torch.cuda.synchronize()
        free, total = torch.cuda.mem_get_info()
        c.mem_budget_bytes = bench.device_budget(c, total, m)
        text = gp.profile_text(c, times=times)
        plan = ex.plan_for(text, 0, "heu")
        pj = json.loads(plan["plan_json"])
        e = ex.Executor(text, plan["timeline"], ex.make_config(c, plan["layers_per_stage"]))
        tok, lab = ex.synthetic_batch(c)
        ms = []
        for _ in range(6):
            t0 = time.perf_counter()
            e.step(tok, lab)
            r = e.report()
            ms.append((round(r["iteration_ms"], 1), round((time.perf_counter() - t0) * 1000, 1)))
        print(f"margin {m}: S={pj['S']} peak={int(pj['peak_bytes'])/1e9:.1f}GB pool_hw={r['pool_high_water_bytes']/1e9:.1f}GB "
              f"exposed={r['exposed_recompute_ms']:.1f} steps(dev,wall)={ms}", flush=True)
        e.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
