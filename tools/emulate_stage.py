"""One TP rank of each TP·PP stage on one B200 (default: the 7B TP2·PP4 headline): exposed
recompute with the plan's comm windows. CLI over paper_2406_08756_b200/stage_emulation.py.

The headline configuration (GPT-7B, micro-batch 32, TP2·PP4, 8 microbatches) needs eight GPUs;
gpurun has one. This runs each stage's TP-rank-0 executor alone (exec.standalone_stage: pipeline
receives read synthetic activations / gradients, sends are skipped) with every TP all-reduce
replaced by a stand-in kernel (exec.comm_standin_us) that holds the TP stream for the transfer
time the plan's window capacities assume (2(t-1)/t * [T,h] bf16 / NVLINK_BUS_GBS, the profiler's
comm model). The recompute items the plan files into those windows run on the side stream against
it, so window overlap, on-demand recompute and waits are measured on real B200 kernels; the SM and
HBM traffic of a real NCCL all-reduce is not modelled (the stand-in sleeps on 16 CTAs).

Per stage: the HEU plan, the same plan with recompute launches elided (no-recompute floor), and
Megatron full recompute. Writes one JSON document.

    python tools/emulate_stage.py [--model 7b] [--stages 0,1,2,3] [--out profiles/x.json]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2406_08756_b200 import gpt_profile as gp  # noqa: E402
from paper_2406_08756_b200 import profiler  # noqa: E402
from paper_2406_08756_b200 import stage_emulation as se  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--stages", default="0,1,2,3")
    ap.add_argument("--micro-batch", type=int, default=0)
    ap.add_argument("--tp", type=int, default=0, help="default: the model config's (7b: TP2 PP4 M8)")
    ap.add_argument("--pp", type=int, default=0)
    ap.add_argument("--microbatches", type=int, default=0)
    ap.add_argument("--budget-gb", type=float, default=0.0,
                    help="ledger budget per GPU (default: this B200's HBM minus the bench's unmodelled reserve)")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--ctas", type=int, default=16)
    ap.add_argument("--variants", default="heu,elided,full_recompute",
                    help="comma list of heu, elided, full_recompute, selective")
    ap.add_argument("--op-timing", action="store_true", help="per-operator device times of the HEU run")
    ap.add_argument("--window-join", type=int, default=1, help="exec.window_join (1: reference semantics)")
    ap.add_argument("--standin-passes", type=int, default=0,
                    help="exec.comm_standin_passes: the stand-in all-reduce also streams its buffer through HBM "
                         "this many times (the local traffic and SM occupancy of a ring all-reduce; 0: sleep only)")
    ap.add_argument("--out", default="gpurun_out/emulate_tp2pp4.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base = gp.CONFIGS[a.model]
    tp = a.tp or base.tp
    c = gp.GPTConfig(**{**base.__dict__, "tp": tp, "pp": a.pp or base.pp, "vocab": gp.padded_vocab(tp),
                        "n_microbatches": a.microbatches or base.n_microbatches, "dropout": 0.1})
    if a.micro_batch:
        c.micro_batch = a.micro_batch
    t0 = time.perf_counter()
    times = profiler.measure_op_times(c)
    torch.cuda.empty_cache()
    prof_s = time.perf_counter() - t0
    _, total = torch.cuda.mem_get_info()
    c.mem_budget_bytes = int(a.budget_gb * 1e9) if a.budget_gb else bench.device_budget(c, total)
    text = gp.profile_text(c, times=times)
    out = {"workload": f"gpt-{a.model} TP{c.tp}xPP{c.pp}, micro-batch {c.micro_batch}, seq {c.seq}, "
                       f"{c.n_microbatches} microbatches; TP rank 0 of each stage alone on one B200",
           "comm_model": {"standin_us_per_allreduce": round(se.standin_us(c), 3),
                          "nvlink_bus_gbs": profiler.NVLINK_BUS_GBS, "bytes": 2 * c.tokens * c.hidden, "ctas": a.ctas,
                          "standin_passes": a.standin_passes,
                          "note": "stand-in kernel holds the TP stream for the modelled transfer time"
                                  + ("; real NCCL SM/HBM contention not modelled" if not a.standin_passes else
                                     f", streaming its buffer through HBM {a.standin_passes}x (in-place read + write) "
                                     "on the stand-in CTAs: a ring all-reduce's local traffic")},
           "profiler_s": round(prof_s, 2), "ledger_budget_bytes": c.mem_budget_bytes,
           "profile_op_us": {k: float(v) for k, v in times.items()}, "window_join": bool(a.window_join),
           "budget": "reduced (--budget-gb)" if a.budget_gb else "device HBM minus unmodelled reserve",
           "stages": {}}
    for s in (int(x) for x in a.stages.split(",")):
        row = se.emulate(c, text, [s], steps=a.steps, warmup=a.warmup, ctas=a.ctas,
                         variants=tuple(a.variants.split(",")), op_timing=a.op_timing,
                         extra_opts={"window_join": bool(a.window_join),
                                     "comm_standin_passes": a.standin_passes})[str(s)]
        out["stages"][str(s)] = row
        print(json.dumps({"stage": s, "exposed_fraction_of_iteration": row.get("exposed_fraction_of_iteration"),
                          "crosscheck_ms": row.get("crosscheck_ms"),
                          **{f"{k}_ms": row[k].get("iteration_ms") for k in a.variants.split(",") if k in row}}),
              flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
