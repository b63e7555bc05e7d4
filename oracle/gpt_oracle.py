"""TEST INFRASTRUCTURE ONLY — CPU fp32 numerical oracle of the GPT training step.

The reference has no numerics (its operators are names, times and byte counts
in the profile), so loss/gradient parity is *unpinned*
by the reference: this is the builder's own oracle, a plain PyTorch-CPU fp32
restatement of the model the executor runs (Megatron-style pre-LN GPT block,
gpt_profile.py templates): token + position embedding, per layer
LN1 -> QKV -> causal softmax attention -> projection + residual -> LN2 -> FC1
-> tanh-GeLU -> FC2 + residual, final LN, untied LM head, mean token
cross-entropy over all microbatches.

Dropout (hidden dropout on the embedding and on both residual branches; the
attention probabilities are not dropped) uses the executor's masks exactly:
Philox-4x32-10 (Salmon et al., SC'11; the Random123 algorithm, pinned by its
published known-answer vectors in tests/test_oracle.py) keyed by the step seed,
with the counter (group of 8 elements, stream id) and stream ids
  embedding        (0xFFFF << 32) | mb
  attention branch ((layer + 1) << 32) | (mb << 8) | 5
  MLP branch       ((layer + 1) << 32) | (mb << 8) | 11
(layer = global layer index, mb = microbatch of the step), element e of a
[tokens, hidden] tensor drawing the 16-bit half e % 2 of word (e % 8) // 2 of group e // 8,
kept iff the draw is >= floor(p * 2^16); kept values are scaled by 1 / (1 - p) in fp32.
(executor.cpp drop_stream / kEmbedStream, common.cuh keep_bits8.)

Used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

_M0, _M1 = 0xD2511F53, 0xCD9E8D57
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_U32 = np.uint64(0xFFFFFFFF)
EMBED_STREAM = 0xFFFF << 32
SITE_ATTN, SITE_MLP = 5, 11  # Op::PROJ_RES, Op::FC2_RES (runtime/gpt_stage.hpp)


def philox4x32_10(ctr: tuple, key: tuple) -> tuple:
    """Philox-4x32-10 on numpy arrays of uint32 values (held in uint64). ctr = 4 words, key = 2 words."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & _U32 for x in ctr)
    k0, k1 = np.uint64(key[0]) & _U32, np.uint64(key[1]) & _U32
    m0, m1 = np.uint64(_M0), np.uint64(_M1)
    for _ in range(10):
        p0 = m0 * c0
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _U32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _U32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + np.uint64(_W0)) & _U32
        k1 = (k1 + np.uint64(_W1)) & _U32
    return c0, c1, c2, c3


def drop_threshold(p: float) -> int:
    """16-bit keep threshold (common.cuh drop_threshold16)."""
    t = float(np.float32(p)) * 65536.0
    return 65536 if t >= 65536.0 else int(t)


def keep_mask(seed: int, stream: int, n: int, p: float) -> np.ndarray:
    """Bool keep-mask of n consecutive elements of dropout stream `stream` (common.cuh keep_bits8):
    element e draws the 16-bit half e % 2 (low first) of word (e % 8) // 2 of Philox group e // 8."""
    if p <= 0:
        return np.ones(n, dtype=bool)
    groups = np.arange((n + 7) // 8, dtype=np.uint64)
    r = philox4x32_10((groups & _U32, groups >> np.uint64(32), np.full_like(groups, stream & 0xFFFFFFFF),
                       np.full_like(groups, stream >> 32)), (seed & 0xFFFFFFFF, seed >> 32))
    words = np.stack(r, axis=1)                                     # [groups, 4]
    halves = np.stack([words & np.uint64(0xFFFF), words >> np.uint64(16)], axis=2)  # [groups, 4, 2]
    draws = halves.reshape(-1)[:n]
    return draws >= np.uint64(drop_threshold(p))


def step_seed(seed: int, step: int) -> int:
    """Dropout key of training step `step` (1-based), executor.cpp."""
    return seed + step * 1000003


def layer_stream(layer: int, mb: int, site: int) -> int:
    return ((layer + 1) << 32) | (mb << 8) | site


def _t(a: np.ndarray, shape) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float32).reshape(shape), requires_grad=True)


def gpt_step(params: dict[str, np.ndarray], shapes: dict[str, tuple], tokens: np.ndarray, labels: np.ndarray, *,
             n_layers: int, hidden: int, heads: int, seq: int, micro_batch: int, n_micro: int, eps: float = 1e-5,
             dropout: float = 0.0, seed: int = 42, step: int = 1,
             threads: int | None = None) -> tuple[float, dict[str, np.ndarray]]:
    """Returns (mean token loss, fp32 gradients by parameter name) of one training step on the
    UNSHARDED model (parameter names as a TP = 1, PP = 1 executor reports them)."""
    if threads:
        torch.set_num_threads(threads)
    P = {k: _t(v, shapes[k]) for k, v in params.items()}
    D = hidden // heads
    T = micro_batch * seq
    tok = torch.tensor(tokens.reshape(n_micro, T).astype(np.int64))
    lab = torch.tensor(labels.reshape(n_micro, T).astype(np.int64))
    mask = torch.ones(seq, seq, dtype=torch.bool).triu(1)
    key = step_seed(seed, step)
    scale = float(np.float32(1.0) / (np.float32(1.0) - np.float32(dropout))) if dropout > 0 else 1.0

    def drop(x: torch.Tensor, stream: int) -> torch.Tensor:
        if dropout <= 0:
            return x
        keep = torch.from_numpy(keep_mask(key, stream, x.numel(), dropout).reshape(x.shape))
        return torch.where(keep, x * scale, torch.zeros((), dtype=x.dtype))

    total = 0.0
    for m in range(n_micro):
        pos = torch.arange(T) % seq
        x = drop(P["wte"][tok[m]] + P["wpe"][pos], EMBED_STREAM | m)
        for l in range(n_layers):
            p = f"l{l}."
            y = F.layer_norm(x, (hidden,), P[p + "ln1_g"], P[p + "ln1_b"], eps)
            qkv = y @ P[p + "w_qkv"].t() + P[p + "b_qkv"]
            q, k, v = qkv.view(micro_batch, seq, 3, heads, D).permute(2, 0, 3, 1, 4)
            att = (q @ k.transpose(-1, -2)) / math.sqrt(D)
            att = att.masked_fill(mask, float("-inf")).softmax(-1)
            o = (att @ v).permute(0, 2, 1, 3).reshape(T, hidden)
            res1 = x + drop(o @ P[p + "w_proj"].t() + P[p + "b_proj"], layer_stream(l, m, SITE_ATTN))
            y2 = F.layer_norm(res1, (hidden,), P[p + "ln2_g"], P[p + "ln2_b"], eps)
            f1 = y2 @ P[p + "w_fc1"].t() + P[p + "b_fc1"]
            g = F.gelu(f1, approximate="tanh")
            x = res1 + drop(g @ P[p + "w_fc2"].t() + P[p + "b_fc2"], layer_stream(l, m, SITE_MLP))
        yf = F.layer_norm(x, (hidden,), P["lnf_g"], P["lnf_b"], eps)
        logits = yf @ P["w_head"].t()
        loss = F.cross_entropy(logits, lab[m], reduction="sum") / (T * n_micro)
        loss.backward()
        total += float(loss.detach())
    grads = {k: v.grad.numpy().ravel().copy() if v.grad is not None else np.zeros(v.numel(), np.float32)
             for k, v in P.items()}
    return total, grads
