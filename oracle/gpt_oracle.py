"""TEST INFRASTRUCTURE ONLY — CPU fp32 numerical oracle of the GPT training step.

The reference has no numerics (its operators are names, times and byte counts
in the profile), so loss/gradient parity is *unpinned*
by the reference: this is the builder's own oracle, a plain PyTorch-CPU fp32
restatement of the model the executor runs (Megatron-style pre-LN GPT block,
gpt_profile.py templates): token + position embedding, per layer
LN1 -> QKV -> causal softmax attention -> projection + residual -> LN2 -> FC1
-> tanh-GeLU -> FC2 + residual, final LN, untied LM head, mean token
cross-entropy over all microbatches. Dropout is off (p = 0) for parity runs.
Used only by tests/ and bench.py's cpu_baseline leg.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F


def _t(a: np.ndarray, shape) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float32).reshape(shape), requires_grad=True)


def gpt_step(params: dict[str, np.ndarray], shapes: dict[str, tuple], tokens: np.ndarray, labels: np.ndarray, *,
             n_layers: int, hidden: int, heads: int, seq: int, micro_batch: int, n_micro: int, eps: float = 1e-5,
             threads: int | None = None) -> tuple[float, dict[str, np.ndarray]]:
    """Returns (mean token loss, fp32 gradients by parameter name)."""
    if threads:
        torch.set_num_threads(threads)
    P = {k: _t(v, shapes[k]) for k, v in params.items()}
    D = hidden // heads
    T = micro_batch * seq
    tok = torch.tensor(tokens.reshape(n_micro, T).astype(np.int64))
    lab = torch.tensor(labels.reshape(n_micro, T).astype(np.int64))
    mask = torch.ones(seq, seq, dtype=torch.bool).triu(1)
    total = 0.0
    for m in range(n_micro):
        pos = torch.arange(T) % seq
        x = P["wte"][tok[m]] + P["wpe"][pos]
        for l in range(n_layers):
            p = f"l{l}."
            y = F.layer_norm(x, (hidden,), P[p + "ln1_g"], P[p + "ln1_b"], eps)
            qkv = y @ P[p + "w_qkv"].t() + P[p + "b_qkv"]
            q, k, v = qkv.view(micro_batch, seq, 3, heads, D).permute(2, 0, 3, 1, 4)
            att = (q @ k.transpose(-1, -2)) / math.sqrt(D)
            att = att.masked_fill(mask, float("-inf")).softmax(-1)
            o = (att @ v).permute(0, 2, 1, 3).reshape(T, hidden)
            res1 = x + o @ P[p + "w_proj"].t() + P[p + "b_proj"]
            y2 = F.layer_norm(res1, (hidden,), P[p + "ln2_g"], P[p + "ln2_b"], eps)
            f1 = y2 @ P[p + "w_fc1"].t() + P[p + "b_fc1"]
            g = F.gelu(f1, approximate="tanh")
            x = res1 + g @ P[p + "w_fc2"].t() + P[p + "b_fc2"]
        yf = F.layer_norm(x, (hidden,), P["lnf_g"], P["lnf_b"], eps)
        logits = yf @ P["w_head"].t()
        loss = F.cross_entropy(logits, lab[m], reduction="sum") / (T * n_micro)
        loss.backward()
        total += float(loss.detach())
    grads = {k: v.grad.numpy().ravel().copy() if v.grad is not None else np.zeros(v.numel(), np.float32)
             for k, v in P.items()}
    return total, grads
