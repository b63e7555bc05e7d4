"""GPT model configurations and their Lynx profile documents.

The reference's profile is an abstract operator graph (names, times, byte
counts; proj/include/lynx/profile.hpp:27-83). This module emits the profile of
a real Megatron-style GPT block so that the same planner produces plans the
B200 executor can run. Template, per TP rank,
T = micro_batch * seq tokens, bf16 activations:

  TP > 1 (15 ops; comm ops are the TP all-reduce windows CTime_1..4)
    0 ln1  1 qkv  2 attn  3 proj(partial, 0 B)  4 ar1(comm)  5 ln2  6 fc1  7 gelu
    8 fc2(partial, 0 B)  9 ar2(comm, checkpoint)  10 mlp_bwd  11 ar_b1(comm)
    12 attn_bwd  13 ar_b2(comm)  14 ln1_bwd
  TP = 1 (11 ops; no windows — every recompute is on the critical path)
    0 ln1  1 qkv  2 attn  3 proj_res  4 ln2  5 fc1  6 gelu  7 fc2_res(checkpoint)
    8 mlp_bwd  9 attn_bwd  10 ln1_bwd

Times come either from a roofline estimate (`estimate_times`) or from
measurements of the executor's own kernels on B200 (`profiler.py`, the
paper's Fig. 5 profiler role). Static bytes follow the 16 B/parameter model states of
the paper that the executor allocates: bf16 weights and gradients,
fp32 master weights and Adam m, v.
"""
from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from fractions import Fraction

BYTES_PER_PARAM_STATIC = 16  # bf16 param 2 + bf16 grad 2 + fp32 master 4 + m 4 + v 4


@dataclass
class GPTConfig:
    name: str = "gpt-tiny"
    n_layers: int = 4
    hidden: int = 512
    heads: int = 8
    seq: int = 256
    micro_batch: int = 2
    vocab: int = 50304
    tp: int = 1
    pp: int = 1
    n_microbatches: int = 1
    dropout: float = 0.1
    mem_budget_bytes: int = 0  # 0 -> derive from device capacity
    comm_scale: str = "1"
    # Use the tensor-parallel template (with its four all-reduce windows) even at tp = 1;
    # the executor then runs the all-reduces on a one-rank communicator. Window times are
    # modelled for tp_model ranks so the planner has windows to fill.
    tp_template: bool = False
    tp_model: int = 2

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def tokens(self) -> int:
        return self.micro_batch * self.seq

    @property
    def vocab_parallel(self) -> bool:
        """Megatron vocab-parallel LM head + cross-entropy: TP > 1 and the vocabulary padded to 128 * tp
        rows (runtime/gpt_stage.hpp ModelCfg::vocab_parallel); otherwise the head is replicated."""
        return self.tp > 1 and self.vocab % (128 * self.tp) == 0

    def layer_params(self) -> int:
        h = self.hidden
        return 12 * h * h + 13 * h

    def params(self) -> int:
        h = self.hidden
        return self.n_layers * self.layer_params() + self.vocab * h * 2 + self.seq * h + 2 * h

    def flops_per_token(self) -> float:
        """Model FLOPs per token, fwd + bwd, no recompute (Megatron count)."""
        L, h, s, V = self.n_layers, self.hidden, self.seq, self.vocab
        return 72.0 * L * h * h + 12.0 * L * s * h + 6.0 * h * V


def padded_vocab(tp: int, vocab: int = 50257) -> int:
    """GPT-2's 50257 tokens padded to a multiple of 128 * tp: every TP rank then holds an
    equal, 128-aligned slice of the vocab-parallel LM head (50304 at TP1, 50432 at TP2, 50688 at TP4,
    51200 at TP8)."""
    m = 128 * tp
    return (vocab + m - 1) // m * m


CONFIGS = {
    "tiny": GPTConfig("gpt-tiny", 4, 512, 8, 256, 2, 50304, 1, 1, 1),
    "1.3b": GPTConfig("gpt-1.3b", 32, 1792, 16, 2048, 16, 50304, 2, 4, 8),
    "7b": GPTConfig("gpt-7b", 32, 4096, 32, 2048, 32, 50304, 2, 4, 8),
    "13b": GPTConfig("gpt-13b", 40, 5120, 40, 2048, 8, 50304, 4, 2, 8),
    "20b": GPTConfig("gpt-20b", 44, 6144, 64, 2048, 8, 50304, 8, 1, 8),
}


def op_bytes(c: GPTConfig) -> dict[str, int]:
    T, h, t = c.tokens, c.hidden, c.tp
    hp = h // t
    return {
        "ln": 2 * T * h + 8 * T,
        "qkv": 2 * T * 3 * hp,
        "attn": 2 * T * hp + 4 * c.micro_batch * (c.heads // t) * c.seq,
        "act": 2 * T * h,
        "fc1": 2 * T * 4 * hp,
        "embed": 2 * T * h,
        "head": 4 * T,
    }


def estimate_times(c: GPTConfig, gemm_tflops: float = 1200.0, attn_tflops: float = 450.0, hbm_gbs: float = 6000.0,
                   nvlink_gbs: float = 700.0) -> dict[str, Fraction]:
    """Roofline estimate of each template op's time in µs (integer ns resolution)."""
    T, h, t, s, b = c.tokens, c.hidden, c.tp, c.seq, c.micro_batch
    hp = h // t

    def g(m, n, k):
        return 2.0 * m * n * k / (gemm_tflops * 1e6)

    def mem(nbytes):
        return nbytes / (hbm_gbs * 1e3)

    tw = c.tp_model if (c.tp == 1 and c.tp_template) else t

    def ar(nbytes):
        return 0.0 if tw == 1 else 2.0 * (tw - 1) / tw * nbytes / (nvlink_gbs * 1e3)

    attn_f = 2.0 * b * (c.heads // t) * s * s * (h // c.heads) / (attn_tflops * 1e6)  # causal: QK^T + PV halves
    est = {
        "ln1": mem(4 * T * h),
        "qkv": g(T, 3 * hp, h),
        "attn": attn_f,
        "proj": g(T, h, hp),
        "ar1": ar(2 * T * h) + mem(6 * T * h),
        "proj_res": g(T, h, hp) + mem(6 * T * h),
        "ln2": mem(4 * T * h),
        "fc1": g(T, 4 * hp, h),
        "gelu": mem(4 * T * 4 * hp),
        "fc2": g(T, h, 4 * hp),
        "ar2": ar(2 * T * h) + mem(6 * T * h),
        "fc2_res": g(T, h, 4 * hp) + mem(6 * T * h),
        "mlp_bwd": 2 * (g(T, 4 * hp, h) + g(T, h, 4 * hp)) + mem(12 * T * 4 * hp),
        "ar_b1": ar(2 * T * h),
        "attn_bwd": 2 * (g(T, 3 * hp, h) + g(T, h, hp)) + 3.5 * attn_f + mem(12 * T * h),
        "ar_b2": ar(2 * T * h),
        "ln1_bwd": mem(8 * T * h),
        "embed": mem(6 * T * h),
        "final_ln": mem(4 * T * h),
        "lm_head": 3 * g(T, c.vocab, h) + mem(6 * T * c.vocab),
    }
    return {k: Fraction(round(v * 1000), 1000) for k, v in est.items()}


def _op(i, name, kind, time_us: Fraction, out_bytes, deps):
    t = time_us.numerator if time_us.denominator == 1 else f"{time_us.numerator}/{time_us.denominator}"
    return {"id": i, "name": name, "kind": kind, "time_us": t, "out_bytes": int(out_bytes), "deps": deps}


def layer_template(c: GPTConfig, times: dict[str, Fraction]) -> dict:
    B = op_bytes(c)
    if c.tp > 1 or c.tp_template:
        spec = [
            ("ln1", "compute", B["ln"], []), ("qkv", "compute", B["qkv"], [0]), ("attn", "compute", B["attn"], [1]),
            ("proj", "compute", 0, [2]), ("ar1", "comm", B["act"], [3]), ("ln2", "compute", B["ln"], [4]),
            ("fc1", "compute", B["fc1"], [5]), ("gelu", "compute", B["fc1"], [6]), ("fc2", "compute", 0, [7]),
            ("ar2", "comm", B["act"], [4, 8]), ("mlp_bwd", "compute", B["act"], [5, 6, 7]),
            ("ar_b1", "comm", B["act"], [10]), ("attn_bwd", "compute", B["act"], [0, 1, 2, 4, 5, 11]),
            ("ar_b2", "comm", B["act"], [12]), ("ln1_bwd", "compute", B["act"], [0, 13]),
        ]
        ops = [_op(i, n, k, times[n], b, d) for i, (n, k, b, d) in enumerate(spec)]
        return {"ops": ops, "fwd_comm_ids": [4, 9], "bwd_comm_ids": [11, 13], "checkpoint_id": 9}
    spec = [
        ("ln1", B["ln"], []), ("qkv", B["qkv"], [0]), ("attn", B["attn"], [1]), ("proj_res", B["act"], [2]),
        ("ln2", B["ln"], [3]), ("fc1", B["fc1"], [4]), ("gelu", B["fc1"], [5]), ("fc2_res", B["act"], [3, 6]),
        ("mlp_bwd", B["act"], [4, 5, 6]), ("attn_bwd", B["act"], [0, 1, 2, 3, 4, 8]), ("ln1_bwd", B["act"], [0, 9]),
    ]
    ops = [_op(i, n, "compute", times[n], b, d) for i, (n, b, d) in enumerate(spec)]
    return {"ops": ops, "fwd_comm_ids": [], "bwd_comm_ids": [], "checkpoint_id": 7}


def profile(c: GPTConfig, times: dict[str, Fraction] | None = None, device_bytes: int | None = None,
            reserve_bytes: int = 0) -> dict:
    """Profile document for config `c`. mem_budget_bytes = c.mem_budget_bytes if set, else
    device_bytes - reserve_bytes (transient workspace the ledger does not model)."""
    times = times or estimate_times(c)
    B = op_bytes(c)
    budget = c.mem_budget_bytes or ((device_bytes or 180_000_000_000) - reserve_bytes)
    static = BYTES_PER_PARAM_STATIC * (c.params() // 1)  # whole model; stages take static * L_s / L
    static = static // c.tp
    return {
        "model": {
            "name": c.name,
            "n_layers": c.n_layers,
            "static_bytes": int(static),
            "layer": layer_template(c, times),
            "embed_ops": [_op(0, "embed", "compute", times["embed"], B["embed"], [])],
            "head_ops": [_op(0, "final_ln", "compute", times["final_ln"], B["ln"], []),
                         _op(1, "lm_head", "compute", times["lm_head"], B["head"], [0])],
        },
        "hardware": {"mem_budget_bytes": int(budget), "comm_scale": c.comm_scale},
        "pipeline": {"n_stages": c.pp, "n_microbatches": c.n_microbatches, "schedule_kind": "1f1b"},
    }


def profile_text(c: GPTConfig, **kw) -> str:
    return json.dumps(profile(c, **kw), indent=1)


def config_dict(c: GPTConfig) -> dict:
    d = asdict(c)
    d["head_dim"] = c.head_dim
    return d
