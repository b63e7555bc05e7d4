"""Benchmark: GPT training tokens/s with a Lynx HEU recompute plan on B200; exposed recompute ms/iter.

Metric (BASELINE.json): "GPT-7B train tokens/s, 8xB200 TP2·PP4; exposed recompute ms/iter".
One step = one full training iteration (all microbatches' 1F1B passes, the
plan's recomputation, AdamW) executed by the native executor through the C-ABI.

  python bench.py                                  # N=1: GPT-7B, TP1 PP1, mb 32, seq 2048, HEU plan
  python -m torch.distributed.run --nproc-per-node N bench.py --gpus N   # N in {2,4,8}: TP2 x PP(N/2)
  python bench.py --impl reference                 # CPU reference arm (host cores)

At N=1 the metric's own model (GPT-7B, mb 32, s 2048) is run whole on one
B200: 6.7 B parameters (120 GB of weights + fp32 master/grad/Adam state) leave
~55 GB for activations, so retain-all OOMs and the HEU plan decides what to
recompute. With TP = 1 there are no all-reduce windows, so all recomputation is
exposed on the critical path; the baselines (retain-all, full recompute) are
reported beside it (--baselines).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GPT-7B train tokens/s, 8×B200 TP2·PP4; exposed recompute ms/iter"


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


from paper_2406_08756_b200.clocks import ClockSampler  # noqa: E402  (NVML clocks during the timed region)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_for(n_gpus: int, args):
    from paper_2406_08756_b200 import gpt_profile as gp
    base = gp.CONFIGS[args.model]
    if n_gpus == 1:
        tp, pp, m = 1, 1, args.microbatches or 1
    else:
        tp = 2
        pp = n_gpus // 2
        m = args.microbatches or max(2 * pp, 2)
    c = gp.GPTConfig(**{**base.__dict__, "tp": tp, "pp": pp, "n_microbatches": m, "dropout": 0.1,
                        "vocab": gp.padded_vocab(tp)})
    if args.micro_batch:
        c.micro_batch = args.micro_batch
    return c


def device_budget(c, device_bytes: int, margin_gib: float = 8.0) -> int:
    """Ledger budget = HBM minus what the ledger does not model (runtime scratch, transients, context)."""
    T, h = c.tokens, c.hidden
    hp = h // c.tp
    # + fp32 LM-head and embedding gradient accumulators (last / first stage; both at PP = 1)
    scratch = 2 * T * h * 3 + 2 * T * 4 * hp + 4096 * c.vocab * 2 + 64 * 2**20 + 4 * c.vocab * h * 2 + 4 * c.seq * h
    transients = 2 * T * h * 6 + 4 * T * h + (2 * T * h + 8 * T)  # grads in flight, embed ws, head dy/ln_f
    # HEU's peak (heusched.cpp:260-277) counts retained tensors only; one layer's
    # discarded tensors are physically alive while that layer runs.
    one_layer = (2 * T * h + 8 * T) * 2 + 2 * T * 3 * hp + 2 * T * hp + 2 * T * h * 2 + 2 * T * 4 * hp * 2
    # CUDA context, NCCL buffers and stream-ordered-pool fragmentation: at 7B mb32 the pool was
    # measured holding ~10 GB reserved-but-unusable next to the ledger's activations (a plan with
    # ledger peak 161.6 GB OOMed with 69.6 GB reserved / 59.7 GB used).
    context = int(margin_gib * 2**30)
    return int(device_bytes - scratch - transients - one_layer - context)


def plan_all(c, profile_text: str, baseline: str):
    from paper_2406_08756_b200 import executor as ex
    t0 = time.perf_counter()
    plans = [ex.plan_for(profile_text, s, baseline) for s in range(c.pp)]
    return plans, time.perf_counter() - t0


def cpu_sample_step(c):
    """One bounded-sample step of the CPU numerical port (oracle/gpt_oracle.py): fwd + bwd of ONE GPT
    block of the workload's width and sequence length + the LM head at micro-batch 1, all host cores.
    Returns (seconds, tokens of the sample, model-FLOP scale to the whole workload)."""
    import numpy as np

    from oracle import gpt_oracle
    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    s = gp.GPTConfig("sample", 1, c.hidden, c.heads, c.seq, 1, c.vocab, 1, 1, 1, dropout=0.0)
    shapes = ex.param_shapes(s, 1, True, True)
    rng = np.random.default_rng(0)
    params = {k: (rng.standard_normal(int(np.prod(v))) * 0.02).astype(np.float32) for k, v in shapes.items()}
    for k in shapes:
        if k.endswith("_g"):
            params[k][:] = 1.0
    tok, lab = ex.synthetic_batch(s)
    t0 = time.perf_counter()
    gpt_oracle.gpt_step(params, shapes, tok, lab, n_layers=1, hidden=s.hidden, heads=s.heads, seq=s.seq,
                        micro_batch=1, n_micro=1)
    return time.perf_counter() - t0, s.tokens, s.flops_per_token() / c.flops_per_token()


def cpu_baseline(c, budget_s: float = 20.0) -> dict:
    """The CPU numerical port (oracle/gpt_oracle.py) on host cores, on a bounded sample of the
    workload (one GPT block of the same width and sequence length + LM head, micro-batch 1),
    scaled to the whole model by model FLOPs per token."""
    import numpy as np
    import torch

    from oracle import gpt_oracle
    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    s = gp.GPTConfig("sample", 1, c.hidden, c.heads, c.seq, 1, c.vocab, 1, 1, 1, dropout=0.0)
    shapes = ex.param_shapes(s, 1, True, True)
    rng = np.random.default_rng(0)
    params = {k: (rng.standard_normal(int(np.prod(v))) * 0.02).astype(np.float32) for k, v in shapes.items()}
    for k in shapes:
        if k.endswith("_g"):
            params[k][:] = 1.0
    tok, lab = ex.synthetic_batch(s)
    n, t_total = 0, 0.0
    while t_total < budget_s and n < 3:
        t0 = time.perf_counter()
        gpt_oracle.gpt_step(params, shapes, tok, lab, n_layers=1, hidden=s.hidden, heads=s.heads, seq=s.seq,
                            micro_batch=1, n_micro=1)
        t_total += time.perf_counter() - t0
        n += 1
    sample_tokens_s = n * s.tokens / t_total
    scaled = sample_tokens_s * s.flops_per_token() / c.flops_per_token()
    return {"value": scaled, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"torch-CPU fp32 fwd+bwd of 1 GPT block (h={c.hidden}, s={c.seq}, mb=1) + LM head, "
                      f"{n} step(s) in {t_total:.1f}s = {sample_tokens_s:.1f} tok/s, scaled by model FLOPs/token "
                      f"({s.flops_per_token():.3g} -> {c.flops_per_token():.3g})"}


def reference_simulate(c, profile_text: str) -> dict | None:
    """The reference's own CPU executor simulate() on the same profile (oracle/_ref), 1 core."""
    try:
        from oracle import ref as oref
        if not oref.available():
            return None
        R = oref.RefLib()
        t0 = time.perf_counter()
        out = json.loads(R.simulate(profile_text, None, "0", 0, 10000))
        wall = time.perf_counter() - t0
        return {"wall_s": round(wall, 4), "predicted_iteration_us": out["iteration_us"],
                "memory_peaks": out["memory_peaks"], "cores": 1}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def reference_planner(total_bytes: int, model: str) -> dict | None:
    """SURVEY §8d CPU item 1: the reference planner (shim-built lynx_core, oracle/_ref) on the
    headline TP2xPP4 profile: search_partition plus the HEU stage plans, single-threaded, beside
    this repo's native planner on the same text (outputs must be identical)."""
    try:
        from oracle import ref as oref
        from paper_2406_08756_b200 import gpt_profile as gp
        from paper_2406_08756_b200 import planner
        if not oref.available():
            return None
        c = gp.GPTConfig(**{**gp.CONFIGS[model].__dict__, "tp": 2, "pp": 4, "n_microbatches": 8, "dropout": 0.1})
        c.mem_budget_bytes = device_budget(c, total_bytes)
        text = gp.profile_text(c)
        R = oref.RefLib()
        t0 = time.perf_counter()
        ref_part = R.partition(text, 10000)
        ref_plans = [R.stage_plan(text, s, None, 10000) for s in range(c.pp)]
        t_ref = time.perf_counter() - t0
        t0 = time.perf_counter()
        our_part = planner.partition_text(text)
        our_plans = [planner.stage_plan_text(text, s) for s in range(c.pp)]
        t_our = time.perf_counter() - t0
        same = json.loads(ref_part) == json.loads(our_part) and all(
            json.loads(a["plan_json"]) == json.loads(b["plan_json"]) for a, b in zip(ref_plans, our_plans))
        return {"profile": f"gpt-{model} TP2xPP4 M=8", "reference_s": round(t_ref, 4), "native_s": round(t_our, 4),
                "identical_outputs": same, "cores": 1,
                "paper_s": "HEU 0.15 s / partition 1.27 s with Gurobi (PAPER.md:1333)"}
    except Exception as e:  # pragma: no cover
        return {"error": str(e).splitlines()[0][:200]}


def load_op_times(path: str) -> dict:
    """Operator times (µs, exact decimal Fractions) of an earlier run — a bench JSON line or a flat
    {op: us} map — so a profiled run (ncu serialises and slows every kernel) plans exactly as the
    measured run did."""
    with open(path) as f:
        doc = json.load(f)
    doc = doc.get("recompute", {}).get("op_times_us", doc)
    return {k: Fraction(str(v)) for k, v in doc.items()}


def run_reference_arm(args):
    """The reference arm: the CPU implementation of the training step (oracle/gpt_oracle.py; the reference
    itself only simulates the step, proj/src/pipesim.cpp) on this host's cores. Each step is one bounded
    sample of the workload — fwd + bwd of one GPT block + LM head at micro-batch 1 — timed on the wall
    clock, so --steps K of them take K x ms_per_step; `value` is that throughput scaled to the whole
    workload by model FLOPs per token. The reference's own simulate() runs beside it (its prediction)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import torch
    from paper_2406_08756_b200 import gpt_profile as gp
    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    c = config_for(max(args.gpus, 1), args)
    c.mem_budget_bytes = 170_000_000_000
    text = gp.profile_text(c)
    for _ in range(args.warmup):  # W warm-up samples, as the GPU arm (~3 s each on 16 cores)
        cpu_sample_step(c)
    secs, toks, scale = [], 0, 1.0
    for _ in range(args.steps):
        dt, toks, scale = cpu_sample_step(c)
        secs.append(dt)
    sample_ms = 1000.0 * statistics.mean(secs)
    value = toks / (sample_ms / 1000.0) * scale
    sample = (f"one step = torch-CPU fp32 fwd+bwd of 1 GPT block (h={c.hidden}, s={c.seq}, micro-batch 1) + LM head "
              f"({toks} tokens, {sample_ms:.0f} ms on {threads} threads); value scaled to {c.name} by model "
              f"FLOPs/token (x{scale:.4g})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "ms_per_step": sample_ms, "config": workload_config(c, args), "dtype": "f32", "data": "synthetic",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_simulate": reference_simulate(c, text), "vs_baseline": None}
    print(json.dumps(line), flush=True)


def workload_config(c, args) -> dict:
    return {"workload": f"{c.name} training step (BASELINE configs[2] shape), seq {c.seq}, micro-batch "
                        f"{c.micro_batch}, {c.n_microbatches} microbatch(es)/iter, TP{c.tp}xPP{c.pp}, "
                        f"{args.plan.upper()} recompute plan",
            "layers": c.n_layers, "hidden": c.hidden, "heads": c.heads, "seq": c.seq, "micro_batch": c.micro_batch,
            "n_microbatches": c.n_microbatches, "tokens_per_step": c.micro_batch * c.seq * c.n_microbatches,
            "parallelism": f"tp{c.tp}pp{c.pp}", "plan": args.plan,
            "l2": "activations are GBs per op (> 126 MB L2); no flush needed"}


def gemm_roofline(c, peaks: dict) -> dict:
    """Dominant kernel: the FC1 forward tcgen05 GEMM at this workload's shape, timed standalone with CUDA
    events on the launching (torch current) stream right after the timed region."""
    import torch

    from paper_2406_08756_b200 import ops
    T, h = c.tokens, c.hidden
    hp = h // c.tp
    a = torch.randn(T, h, device="cuda").bfloat16()
    b = torch.randn(4 * hp, h, device="cuda").bfloat16()
    out = torch.empty(T, 4 * hp, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        ops.gemm(a, b, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    n = 10
    s.record()
    for _ in range(n):
        ops.gemm(a, b, out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    flops = 2.0 * T * 4 * hp * h
    ach = flops / ms / 1e9
    peak = peaks.get("bf16_tflops", 1590.0)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            traffic = json.load(f).get("fc1_fwd_bytes_per_launch")
    except Exception:
        pass
    del a, b, out
    torch.cuda.empty_cache()
    return {"bound": "tensor", "kernel": "gemm_tcgen05 fc1 fwd", "shape": [T, 4 * hp, h], "ms_per_launch": ms,
            "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
            "peak_kind": "measured burst bf16 (MEASURED_PEAKS.json)", "traffic": traffic,
            "flops_per_launch": flops}


def stage_emulation_summary(args, device_total: int) -> dict:
    """The headline TP2xPP4 configuration's stage 0 (four microbatches in flight, the most
    recompute) as TP rank 0 alone on this B200, all-reduces replaced by stand-in kernels that hold
    the TP stream for the modelled transfer time (paper_2406_08756_b200/stage_emulation.py): the
    exposed recompute with the plan's comm windows, against the same plan with recompute elided."""
    import torch

    from paper_2406_08756_b200 import gpt_profile as gp
    from paper_2406_08756_b200 import profiler
    from paper_2406_08756_b200 import stage_emulation as se
    try:
        torch.cuda.empty_cache()
        c2 = config_for(8, args)
        times2 = profiler.measure_op_times(c2) if args.profile == "measured" else None
        torch.cuda.empty_cache()
        c2.mem_budget_bytes = device_budget(c2, device_total, args.mem_margin_gib)
        text2 = gp.profile_text(c2, times=times2)
        row = se.emulate(c2, text2, [0], variants=("heu", "elided"))["0"]
        h, el = row["heu"], row["elided"]
        return {"config": f"stage 0 of {c2.name} TP{c2.tp}xPP{c2.pp}, micro-batch {c2.micro_batch}, "
                          f"{c2.n_microbatches} microbatches ({row['layers_per_stage'][0]} layers + embedding), TP "
                          "rank 0 alone on this B200; PP receives synthetic, each preceded by the stall the "
                          "simulator predicts for this stage (stand-in kernel); each TP all-reduce a stand-in "
                          f"kernel holding the TP stream {se.standin_us(c2):.1f} us (2(t-1)/t [T,h] bf16 at "
                          f"{profiler.NVLINK_BUS_GBS:g} GB/s; NCCL SM/HBM contention not modelled)",
                "plan": row["plan"], "iteration_ms": round(h["iteration_ms"], 3),
                "exposed_recompute_ms": round(h["exposed_recompute_ms"], 3),
                "exposed_fraction_of_iteration": row["exposed_fraction_of_iteration"],
                "recompute_overlapped_ms": round(h["recompute_overlapped_ms"], 3),
                "elided_iteration_ms": round(el["iteration_ms"], 3), "crosscheck_ms": row["crosscheck_ms"],
                "exposed_fraction_of_recompute": row["exposed_fraction_of_recompute"],
                "pipeline_stall_ms": round(sum(row["grad_wait_us"]) / 1000.0, 3),
                "simulated_busy_ms": round(float(row["simulated_period_us"]) * c2.n_microbatches / 1000.0, 3)}
    except Exception as err:  # reported, never fatal for the headline line
        return {"error": str(err).splitlines()[0][:200]}


def tiny_config_line() -> dict:
    """BASELINE configs[0] (tiny GPT, 4 layers, h 512, s 256, micro-batch 2; 8 microbatches per iteration,
    HEU plan, TP1 PP1) through the same executor: tokens/s and the host time spent issuing the step."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import host_issue
        from paper_2406_08756_b200 import gpt_profile as gp
        c = gp.GPTConfig("gpt-tiny", 4, 512, 8, 256, 2, 50304, 1, 1, 8, dropout=0.1)
        r = host_issue.measure(c, "heu", {"reserve_pool": False})
        return {"workload": "gpt-tiny (BASELINE configs[0]) 4 layers h512 s256 mb2, 8 microbatches/iter, HEU, TP1PP1",
                **r, "note": "latency-bound (1e3 short kernels per step); the host issues a launch in ~3 us, so "
                             "host_issue_ms < iteration_ms: the GPU, not the host, bounds the step"}
    except Exception as err:  # reported, never fatal for the headline line
        return {"error": str(err).splitlines()[0][:200]}


def run_variants(args, c, text, plans, cfg, tok, lab, tokens_iter, dev_ms, times) -> dict:
    """Same-box comparison runs after the timed region (N=1):
    - "elided": the same plan with every recompute launch skipped (timing only; regenerated
      tensors are left uninitialised) -> T(plan) - T(elided) cross-checks the exposed recompute
      (SURVEY §8d);
    - with --baselines: Megatron full recompute and retain-all at this micro-batch (OOM at 7B mb32),
      and retain-all / HEU at half the micro-batch, where retain-all fits."""
    import torch

    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    # elided: the consumers of skipped regenerations read stand-in buffers filled with bf16 noise (the fill is
    # timed apart and subtracted): stale pool memory made the remaining GEMMs draw less power and run at a
    # higher clock under the 1 kW cap, which had inflated the cross-check by ~30 % (tools/recompute_accounting.py)
    variants = [("elided", c, text, plans[0]["timeline"], {"elide_recompute": True, "elide_fill": True})]
    if args.baselines:
        variants.append(("full", c, text, None, {}))
        variants.append(("selective", c, text, None, {"plan": "selective"}))
        half = gp.GPTConfig(**{**c.__dict__, "micro_batch": max(1, c.micro_batch // 2)})
        half.mem_budget_bytes = c.mem_budget_bytes
        half_text = gp.profile_text(half)  # analytic op times (the measured ones are for micro-batch c)
        for base in ("retain_all", "heu"):
            variants.append((f"{base}_mb{half.micro_batch}", half, half_text, None, {"plan": base}))
        variants.append(("retain_all", c, text, None, {}))  # expected OOM at 7B mb32: run last
    out = {}
    for name, cc, tt, timeline, opts in variants:
        be, bp = None, None
        try:
            plan_kind = opts.pop("plan", None) or (name if name in ("full", "retain_all", "selective") else "heu")
            if timeline is None:
                bp, _ = plan_all(cc, tt, plan_kind)
                timeline = bp[0]["timeline"]
            ccfg = ex.make_config(cc, [cc.n_layers], exec_opts={"trace": False, **opts})
            btok, blab = ex.synthetic_batch(cc)
            torch.cuda.synchronize()
            free_b = torch.cuda.mem_get_info()[0]
            be = ex.Executor(tt, timeline, ccfg)
            for _ in range(3):  # the first steps grow the stream-ordered pool
                be.step(btok, blab)
            reps = []
            for _ in range(3):  # the median of three steps (one slow step must not decide the cross-check)
                be.step(btok, blab)
                reps.append(be.report())
            for r in reps:
                r["iteration_ms"] -= r.get("elide_fill_ms", 0.0)
            br = sorted(reps, key=lambda r: r["iteration_ms"])[1]
            tok_i = cc.tokens * cc.n_microbatches
            out[name] = {"iteration_ms": round(br["iteration_ms"], 3), "elide_fill_ms": round(br.get("elide_fill_ms", 0.0), 3),
                         "exposed_recompute_ms": round(br["exposed_recompute_ms"], 3),
                         "tokens_per_s": round(tok_i / (br["iteration_ms"] / 1000.0), 1),
                         "micro_batch": cc.micro_batch, "recompute_launches": br["recompute_launches"],
                         "pool_high_water_bytes": br["pool_high_water_bytes"], "free_bytes_before": free_b,
                         "loss": br["loss"], "step_ms_each": [round(r["iteration_ms"], 1) for r in reps]}
            if bp is not None:
                out[name]["plan_peak_bytes"] = json.loads(bp[0]["plan_json"])["peak_bytes"]
            if name == "elided":
                out[name]["exposed_recompute_crosscheck_ms"] = round(dev_ms - br["iteration_ms"], 3)
        except Exception as err:
            out[name] = {"error": str(err).splitlines()[0][:200], "micro_batch": cc.micro_batch}
            if bp is not None:
                out[name]["plan_peak_bytes"] = json.loads(bp[0]["plan_json"])["peak_bytes"]
        finally:
            if be is not None:
                be.close()
    return out


def run_gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_08756_b200 import executor as ex
    from paper_2406_08756_b200 import gpt_profile as gp
    ws, rank, local = dist_env()
    n = max(args.gpus, ws)
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("gloo", init_method="env://")
    c = config_for(n, args)
    from paper_2406_08756_b200._native import lib
    lib().lynx_op_gemm_mode(args.gemm_mode)
    peaks = measured_peaks()
    roof = gemm_roofline(c, peaks) if rank == 0 else None  # before the executor owns the HBM
    times, prof_s = None, 0.0
    if args.op_times:
        times = load_op_times(args.op_times)
    elif args.profile == "measured":
        # B200-measured operator times drive the plan; rank 0 measures and
        # broadcasts so that every rank plans from the same profile document.
        from paper_2406_08756_b200 import profiler
        t0 = time.perf_counter()
        times = profiler.measure_op_times(c) if rank == 0 else None
        torch.cuda.empty_cache()  # the profiler's tensors (~5 GB at 7B) go back to the device for the executor
        if ws > 1:
            obj = [times]
            dist.broadcast_object_list(obj, src=0)
            times = obj[0]
        prof_s = time.perf_counter() - t0
    free, total = torch.cuda.mem_get_info()
    # Memory margin ladder: a plan whose physical footprint (ledger + per-layer transients + pool
    # fragmentation) overflows HBM fails with LYNX_E_OOM in the first warm-up step; at N = 1 the
    # bench then re-plans with a larger margin (recorded in the JSON line as memory.oom_retries).
    margins = [args.mem_margin_gib] + ([m for m in (12.0, 16.0) if m > args.mem_margin_gib] if ws == 1 else [])
    oom_retries = []
    c.mem_budget_bytes = device_budget(c, total, margins[0])
    text = gp.profile_text(c, times=times)
    plans, plan_s = plan_all(c, text, args.plan)
    layers = plans[0]["layers_per_stage"]
    stage, tp_rank = rank // c.tp, rank % c.tp
    nccl_id = ""
    if ws > 1:
        obj = [ex.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    cfg = ex.make_config(c, layers, tp_rank=tp_rank, world_rank=rank, world_size=ws, nccl_id=nccl_id,
                         exec_opts={"trace": False, "probe_fc1": True})
    tok, lab = ex.synthetic_batch(c)
    first, last = stage == 0, stage == c.pp - 1
    sampler = ClockSampler(local)  # NVML initialised before the warm-up, polled only in the timed region
    for mi, margin in enumerate(margins):
        e = None
        try:
            if mi > 0:
                c.mem_budget_bytes = device_budget(c, total, margin)
                text = gp.profile_text(c, times=times)
                plans, plan_s = plan_all(c, text, args.plan)
            e = ex.Executor(text, plans[stage]["timeline"], cfg)
            for _ in range(args.warmup):
                e.step(tok if first else None, lab if last else None)
            break
        except ex.LynxError as err:
            if err.code != 7 or mi + 1 == len(margins):
                raise
            oom_retries.append({"margin_gib": margin, "plan_S": json.loads(plans[stage]["plan_json"])["S"],
                                "error": str(err)[:160]})
            if e is not None:
                e.close()
            torch.cuda.empty_cache()
    # ---- timed region: K steps through the C-ABI with host buffers
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    step_ms, losses, reports = [], [], []
    with sampler as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            losses.append(e.step(tok if first else None, lab if last else None))
            r = e.report()
            reports.append(r)
            step_ms.append(r["iteration_ms"])
        wall = time.perf_counter() - t0
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    dev_ms = float(np.mean(step_ms))
    wall_ms = 1000.0 * wall / args.steps
    exposed = float(np.mean([r["exposed_recompute_ms"] for r in reports]))
    if ws > 1:
        t = torch.tensor([dev_ms, wall_ms, exposed], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, wall_ms, exposed = t.tolist()
    tokens_iter = c.tokens * c.n_microbatches
    value = tokens_iter / (dev_ms / 1000.0)
    e2e = tokens_iter / (wall_ms / 1000.0)
    rep = reports[-1]
    plan0 = json.loads(plans[stage]["plan_json"])
    extra = {}
    if rank == 0 and ws == 1 and (args.baselines or not args.no_crosscheck):
        e.close()
        del e
        print(json.dumps({"partial": True, "value": value, "ms": dev_ms, "exposed_ms": exposed,
                          "report": rep}), file=sys.stderr, flush=True)
        extra = run_variants(args, c, text, plans, cfg, tok, lab, tokens_iter, dev_ms, times)
        e = None
    emu = None
    if rank == 0 and ws == 1 and not args.no_stage_emulation:
        if e is not None:
            e.close()
        e = None
        emu = stage_emulation_summary(args, total)
    tiny = tiny_config_line() if rank == 0 and ws == 1 else None
    if rank != 0:
        return
    step_tflops = c.flops_per_token() * tokens_iter / (dev_ms / 1000.0) / 1e12
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dev_ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic tokens, random-init weights",
        "config": workload_config(c, args),
        "exposed_recompute_ms_per_iter": round(exposed, 3),
        # T(plan) - T(same plan, recompute elided, stand-in buffers noise-filled): the exposed cost measured as
        # lost time, including the power-cap clock drop the extra work causes (the span metric above counts
        # on-demand recompute kernels + main-stream waits only)
        "exposed_recompute_crosscheck_ms": (extra or {}).get("elided", {}).get("exposed_recompute_crosscheck_ms"),
        "recompute": {"plan": plan0, "items": len(plans[stage]["timeline"]["items"]),
                      "launches_per_iter": rep["recompute_launches"],
                      "on_demand_ms": rep["recompute_on_demand_ms"], "overlapped_ms": rep["recompute_overlapped_ms"],
                      "wait_on_recompute_ms": rep["wait_on_recompute_ms"], "baselines": extra or None,
                      "profile": ("replayed " + args.op_times) if args.op_times else args.profile, "profiler_s": round(prof_s, 2),
                      "op_times_us": {k: float(v) for k, v in (times or {}).items()}},
        "tp2pp4_stage_emulation": emu,
        "tiny_config": tiny,
        "memory": {"ledger_budget_bytes": c.mem_budget_bytes, "plan_peak_bytes": plan0["peak_bytes"],
                   "margin_gib": margins[len(oom_retries)], "oom_retries": oom_retries,
                   "pool_high_water_bytes": rep["pool_high_water_bytes"],
                   "static_bytes": rep["static_bytes_allocated"], "device_total_bytes": total},
        "loss": [round(x, 5) for x in losses],
        "step_ms_each": [round(x, 1) for x in step_ms],
        "model_tflops_per_gpu": round(step_tflops / n, 1),
        "mfu_vs_sustained": round(step_tflops / n / peaks.get("bf16_tflops_sustained", 1400.0), 4),
        "roofline": roof,
        "e2e": {"value": round(e2e, 1), "unit": "tokens/s",
                "h2d_bytes_per_step": 2 * 4 * tokens_iter if ws == 1 else 4 * tokens_iter,
                "d2h_bytes_per_step": 4 * tokens_iter},
        "gpu_launches": None,
        "clocks": clk.summary(),
        "planner_s": round(plan_s, 3),
    }
    # roofline of the dominant kernel from CUDA events around every FC1 forward GEMM launch inside the
    # timed steps (forward and recompute, on the launching stream); the isolated pre-run measurement is
    # kept beside it
    n_probe = sum(r.get("probe_fc1_launches", 0) for r in reports)
    if roof is not None and n_probe:
        ms_probe = sum(r["probe_fc1_ms"] for r in reports) / n_probe
        iso = {k: roof[k] for k in ("ms_per_launch", "achieved", "frac")}
        ach = roof["flops_per_launch"] / ms_probe / 1e9
        iso["peak"], iso["peak_kind"] = roof["peak"], roof["peak_kind"]
        peak = peaks.get("bf16_tflops_sustained", roof["peak"])  # kernel timed inside a long step
        roof.update({"peak": peak, "peak_kind": "measured sustained bf16 (MEASURED_PEAKS.json; kernel timed inside "
                     "the step)",
                     "ms_per_launch": round(ms_probe, 4), "achieved": round(ach, 1), "frac": round(ach / peak, 4),
                     "launches_timed": n_probe, "measured": "CUDA events on the launching stream around each FC1 "
                     "forward GEMM (fused GeLU epilogue) inside the timed steps", "isolated": iso})
    # kernels of liblynx_b200.so issued inside the timed region (counted at every launch site)
    line["gpu_launches"] = int(sum(r["kernel_launches"] for r in reports))
    if not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = cpu_baseline(c, budget_s=20.0)
        line["reference_simulate"] = reference_simulate(c, text)
        line["reference_planner"] = reference_planner(total, args.model)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="7b")
    ap.add_argument("--micro-batch", type=int, default=0)
    ap.add_argument("--microbatches", type=int, default=0)
    ap.add_argument("--plan", default="heu", choices=["heu", "full", "retain_all", "selective"])
    ap.add_argument("--baselines", action="store_true", help="also time retain-all / full-recompute plans (N=1)")
    ap.add_argument("--gemm-mode", type=int, default=-1, help="lynx_op_gemm_mode (-1 default, 0 single-CTA, 1 pair)")
    ap.add_argument("--profile", default="measured", choices=["measured", "estimated"],
                    help="operator times for the planner: B200-measured (default) or the analytic estimate")
    ap.add_argument("--op-times", default="", help="plan from the op times of an earlier bench JSON line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-crosscheck", action="store_true", help="skip the recompute-elided timing run")
    ap.add_argument("--no-stage-emulation", action="store_true",
                    help="skip the TP2xPP4 stage-0 run with stand-in all-reduces (N=1)")
    ap.add_argument("--mem-margin-gib", type=float, default=8.0,
                    help="HBM held back from the HEU budget for context and pool fragmentation "
                         "(an OOM retries with 12 and 16 GiB)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
