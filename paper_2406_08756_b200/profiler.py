"""GPU profiler: B200-measured operator times for the profile document.

The reference's profile carries per-operator times the paper obtains from a
CUDA-event profiler of the real model (out of the
reference's own scope). `measure_op_times` times the EXECUTOR
itself: an eight-layer standalone stage of the workload's width,
sequence, micro-batch and TP degree runs training steps with exec.op_timing
(CUDA events around every template operator on the main stream), so each op's
time is that of the exact fused kernel sequence the step launches (FC2-dX with
the GeLU backward epilogue, dropout backward with the bias column sum, bf16
weight-gradient epilogues, the residual epilogues) under the step's own
conditions. At TP > 1 every all-reduce is a stand-in kernel holding 16 CTAs
for the modelled transfer time while the stage runs, as in the stage emulation.
Ops the step does not launch alone are timed as the kernel the executor
launches when regenerating them: `fc1` (plain GEMM: a kept GeLU) and `gelu`
(stand-alone kernel: GeLU regenerated from a kept FC1; in the forward both are
one fused GEMM). Op times of the other layer template (TP = 1 fused residual
GEMMs vs TP partial + all-reduce epilogue) come from the isolated kernels.

    times = measure_op_times(cfg)            # {op name: Fraction(µs)}
    profile = gpt_profile.profile(cfg, times=times)

All-reduce ops cannot be timed on one GPU; their time is the measured residual
epilogue plus the NVLink model (2(t-1)/t · bytes / 725 GB/s, the measured
8-rank bus bandwidth in B200_PROFILING.md).
"""
from __future__ import annotations

import math
from fractions import Fraction

import torch

from . import gpt_profile as gp
from . import ops

NVLINK_BUS_GBS = 725.0


def _time(fn, iters: int = 5, warm: int = 2) -> float:
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return 1000.0 * s.elapsed_time(e) / iters  # µs


def measure_op_times(c: gp.GPTConfig, iters: int = 5, method: str = "executor") -> dict[str, Fraction]:
    """{op: µs} for the profile of `c`; method "executor" (default, see the module docstring) or "isolated"
    (each op's kernels launched alone on random operands)."""
    iso = measure_op_times_isolated(c, iters)
    if method == "isolated":
        return iso
    ms = executor_op_times(c)
    out = dict(iso)
    for k in ("qkv", "attn", "mlp_bwd", "attn_bwd", "ln1_bwd", "embed"):
        out[k] = _us(ms[k])
    out["ln1"] = out["ln2"] = out["final_ln"] = _us((ms["ln1"] + ms["ln2"]) / 2)
    if c.tp > 1 or c.tp_template:
        out["proj"], out["fc2"] = _us(ms["proj"]), _us(ms["fc2"])
        tw = c.tp_model if c.tp == 1 else c.tp
        ar_ms = 2.0 * (tw - 1) / tw * (2 * c.tokens * c.hidden) / (NVLINK_BUS_GBS * 1e6)
        out["ar1"] = _us(ar_ms + ms["ar1_epilogue"])
        out["ar2"] = _us(ar_ms + ms["ar2_epilogue"])
    else:
        out["proj_res"], out["fc2_res"] = _us(ms["proj_res"]), _us(ms["fc2_res"])
    out["lm_head"] = _us(max(ms["head_fwd"] + ms["head_bwd"] - (ms["ln1"] + ms["ln2"]) / 2, 1e-6))
    return out


def _us(ms: float) -> Fraction:
    """ms -> µs as an exact Fraction at ns resolution (the profile's rational time_us)."""
    return Fraction(max(1, round(float(ms) * 1e6)), 1000)


def executor_op_times(c: gp.GPTConfig, steps: int = 2, layers: int = 8, warmup: int = 1,
                      micro: int = 1) -> dict[str, float]:
    """Median device time (ms) of each template operator of a `layers`-layer standalone stage of `c`'s
    shapes, `micro` microbatches (retain-all plan, exec.op_timing; all-reduces as stand-ins at TP > 1).
    Eight layers: in a two-layer stage the LM head's GEMMs (tens of ms at the board's power cap) dominate
    the step and the layer ops after them ran ~10 % slower than inside a full stage
    (profiles/r02_profiler_check.json); with eight they match the stage's own per-op times."""
    import statistics

    from . import executor as ex
    from . import stage_emulation as se
    c2 = gp.GPTConfig(**{**c.__dict__, "n_layers": layers, "pp": 1, "n_microbatches": micro,
                         "mem_budget_bytes": 10**15})
    text = gp.profile_text(c2)
    plan = ex.plan_for(text, 0, "retain_all")
    opts = {"standalone_stage": True, "op_timing": True, "reserve_pool": False}
    if c2.tp > 1 or c2.tp_template:
        opts["comm_standin_us"] = max(se.standin_us(c2), 1.0)
    e = ex.Executor(text, plan["timeline"], ex.make_config(c2, plan["layers_per_stage"], exec_opts=opts))
    tok, lab = ex.synthetic_batch(c2)
    try:
        for _ in range(warmup):
            e.step(tok, lab)  # warm-up (pool growth, first launches)
        acc: dict[str, list[float]] = {}
        for _ in range(steps):
            e.step(tok, lab)
            for k, v in e.report()["op_timing_ms"].items():
                acc.setdefault(k, []).extend(v)
    finally:
        e.close()
        torch.cuda.empty_cache()
    return {k: statistics.median(v) for k, v in acc.items()}


def measure_op_times_isolated(c: gp.GPTConfig, iters: int = 5) -> dict[str, Fraction]:
    dev = "cuda"
    T, h, t = c.tokens, c.hidden, c.tp
    hp = h // t
    H = c.heads // t
    D = c.head_dim
    bf = torch.bfloat16
    r = lambda *s: (torch.randn(*s, device=dev) * 0.02).to(bf)  # noqa: E731
    x, y = r(T, h), r(T, h)
    gam, bet = torch.ones(h, device=dev, dtype=bf), torch.zeros(h, device=dev, dtype=bf)
    w_qkv, b_qkv, w_proj, b_proj = r(3 * hp, h), r(3 * hp), r(h, hp), r(h)
    w_fc1, b_fc1, w_fc2, b_fc2 = r(4 * hp, h), r(4 * hp), r(h, 4 * hp), r(h)
    qkv = r(T, 3 * hp)
    fc1 = r(T, 4 * hp)
    attn_o, lse = ops.attention_fwd(qkv, c.micro_batch, c.seq, H, D)
    times: dict[str, float] = {}

    times["ln1"] = times["ln2"] = _time(lambda: ops.layernorm_fwd(x, gam, bet), iters)
    times["qkv"] = _time(lambda: ops.gemm(x, w_qkv, bias=b_qkv), iters)
    times["attn"] = _time(lambda: ops.attention_fwd(qkv, c.micro_batch, c.seq, H, D), iters)
    proj = lambda: ops.gemm(attn_o, w_proj, bias=b_proj if t == 1 else None)  # noqa: E731
    times["proj"] = _time(proj, iters)
    resid = _time(lambda: ops.bias_dropout_residual(y, b_proj, x, c.dropout, 1, 2), iters)
    # TP = 1: the executor runs PROJ_RES / FC2_RES as one GEMM with the residual epilogue
    times["proj_res"] = _time(lambda: ops.gemm_residual(attn_o, w_proj, x, bias=b_proj, p=c.dropout, seed=1,
                                                        stream_id=2), iters)
    times["fc1"] = _time(lambda: ops.gemm(y, w_fc1, bias=b_fc1), iters)
    times["gelu"] = _time(lambda: ops.gelu_fwd(fc1), iters)  # stand-alone (a GeLU recomputed from a kept FC1)
    times["fc2"] = _time(lambda: ops.gemm(fc1, w_fc2, bias=b_fc2 if t == 1 else None), iters)
    times["fc2_res"] = _time(lambda: ops.gemm_residual(fc1, w_fc2, x, bias=b_fc2, p=c.dropout, seed=1, stream_id=3),
                             iters)
    tw = c.tp_model if (t == 1 and c.tp_template) else t
    ar = 0.0 if tw == 1 else 2.0 * (tw - 1) / tw * (2 * T * h) / (NVLINK_BUS_GBS * 1e3)
    times["ar1"] = times["ar2"] = ar + resid
    times["ar_b1"] = times["ar_b2"] = ar

    g_fc2 = torch.zeros(h, 4 * hp, device=dev)
    g_fc1 = torch.zeros(4 * hp, h, device=dev)
    g_b = torch.zeros(max(4 * hp, 3 * hp, h), device=dev)  # bias-gradient accumulator wide enough for every use

    def mlp_bwd():
        d = ops.dropout_bwd(y, c.dropout, 1, 3)
        ops.column_sum_acc(d, g_b[:h])
        ops.gemm(d, fc1, a_mn=True, b_mn=True, out=g_fc2, epi=ops.EPI_ACC_F32)
        dg = ops.gemm(d, w_fc2, b_mn=True)
        df = ops.gelu_bwd(dg, fc1)
        ops.column_sum_acc(df, g_b)
        ops.gemm(df, y, a_mn=True, b_mn=True, out=g_fc1, epi=ops.EPI_ACC_F32)
        ops.gemm(df, w_fc1, b_mn=True)

    times["mlp_bwd"] = _time(mlp_bwd, iters)
    del g_fc2, g_fc1
    g_proj = torch.zeros(h, hp, device=dev)
    g_qkv = torch.zeros(3 * hp, h, device=dev)
    mean = torch.zeros(T, device=dev)
    rstd = torch.ones(T, device=dev)
    gl = torch.zeros(h, device=dev)

    def attn_bwd():
        dres = ops.layernorm_bwd(y, x, gam, mean, rstd, gl, gl, dres=y)
        d = ops.dropout_bwd(dres, c.dropout, 1, 4)
        ops.column_sum_acc(d, gl)
        ops.gemm(d, attn_o, a_mn=True, b_mn=True, out=g_proj, epi=ops.EPI_ACC_F32)
        do = ops.gemm(d, w_proj, b_mn=True)
        dqkv = ops.attention_bwd(qkv, attn_o, do, lse, c.micro_batch, c.seq, H, D)
        ops.column_sum_acc(dqkv, g_b[:3 * hp])
        ops.gemm(dqkv, y, a_mn=True, b_mn=True, out=g_qkv, epi=ops.EPI_ACC_F32)
        ops.gemm(dqkv, w_qkv, b_mn=True)

    times["attn_bwd"] = _time(attn_bwd, iters)
    times["ln1_bwd"] = _time(lambda: ops.layernorm_bwd(y, x, gam, mean, rstd, gl, gl, dres=y), iters)
    del g_proj, g_qkv, fc1
    tok = torch.randint(0, 50257, (T,), device=dev, dtype=torch.int32)
    wte, wpe = r(c.vocab, h), r(c.seq, h)
    times["embed"] = _time(lambda: ops.embedding_fwd(tok, wte, wpe, c.micro_batch, c.seq, c.dropout, 1, 5), iters)
    times["final_ln"] = times["ln1"]
    chunk = min(4096, T)
    w_head = r(c.vocab, h)
    g_head = torch.zeros(c.vocab, h, device=dev)
    logits = torch.empty(chunk, c.vocab, device=dev, dtype=bf)
    lab = torch.randint(0, c.vocab, (chunk,), device=dev, dtype=torch.int32)

    def head():
        for c0 in range(0, T, chunk):
            ops.gemm(x[c0:c0 + chunk], w_head, out=logits)
            ops.xent_fwd_bwd(logits, lab, 1.0)
            ops.gemm(logits, x[c0:c0 + chunk], a_mn=True, b_mn=True, out=g_head, epi=ops.EPI_ACC_F32)
            ops.gemm(logits, w_head, b_mn=True)

    times["lm_head"] = _time(head, max(2, iters // 2))
    del g_head, logits, w_head, wte
    torch.cuda.empty_cache()
    return {k: Fraction(max(1, round(v * 1000)), 1000) for k, v in times.items()}


def measured_profile(c: gp.GPTConfig, device_bytes: int | None = None, reserve_bytes: int = 0) -> tuple[dict, dict]:
    times = measure_op_times(c)
    torch.cuda.empty_cache()  # release the measurement tensors (they die with measure_op_times' frame)
    return gp.profile(c, times=times, device_bytes=device_bytes, reserve_bytes=reserve_bytes), times


def times_json(times: dict[str, Fraction]) -> dict[str, str]:
    return {k: (str(v.numerator) if v.denominator == 1 else f"{v.numerator}/{v.denominator}") for k, v in times.items()}


if __name__ == "__main__":  # pragma: no cover
    import json
    import sys
    cfg = gp.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
    if len(sys.argv) > 2:
        cfg = gp.GPTConfig(**{**cfg.__dict__, "tp": int(sys.argv[2])})
    t = measure_op_times(cfg)
    print(json.dumps({k: float(v) for k, v in t.items()}, indent=1))
    _ = math
