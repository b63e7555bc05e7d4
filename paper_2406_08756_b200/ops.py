"""Torch-tensor convenience wrappers over the operator C-ABI (include/lynx_b200.h).

PyTorch is used only for device memory and the current CUDA stream; every
computation runs in the sm_100a kernels of `_lib/liblynx_b200.so`. These
wrappers exist for the parity tests and the profiler; the executor calls the
kernels directly from C++.
"""
from __future__ import annotations

import torch

from ._native import call, lib

EPI_BF16, EPI_ACC_F32, EPI_F32, EPI_ACC_BF16 = 0, 1, 2, 3


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _s() -> int:
    return torch.cuda.current_stream().cuda_stream


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_mn: bool = False, b_mn: bool = False, out: torch.Tensor | None = None,
         bias: torch.Tensor | None = None, epi: int = EPI_BF16) -> torch.Tensor:
    """C = A_logical @ B_logical^T with A_logical [M,K], B_logical [N,K].

    a_mn=False: `a` is [M,K];  a_mn=True: `a` is [K,M] (A_logical = a.T).
    b_mn=False: `b` is [N,K];  b_mn=True: `b` is [K,N] (B_logical = b.T).
    """
    M, K = (a.shape[1], a.shape[0]) if a_mn else (a.shape[0], a.shape[1])
    N = b.shape[1] if b_mn else b.shape[0]
    if out is None:
        out = torch.empty(M, N, device=a.device, dtype=torch.bfloat16 if epi in (EPI_BF16, EPI_ACC_BF16) else torch.float32)
    call("lynx_op_gemm", a.data_ptr(), a.stride(0), int(a_mn), b.data_ptr(), b.stride(0), int(b_mn), out.data_ptr(),
         out.stride(0), M, N, K, _p(bias), epi, _s())
    return out


def gemm_gelu(a: torch.Tensor, b: torch.Tensor, *, bias: torch.Tensor | None = None):
    """(C, gelu(C)) with C = bf16(a @ b^T + bias): the FC1 GEMM with its GeLU fused (K-major operands)."""
    M, K = a.shape
    N = b.shape[0]
    c = torch.empty(M, N, device=a.device, dtype=torch.bfloat16)
    g = torch.empty_like(c)
    call("lynx_op_gemm_gelu", a.data_ptr(), a.stride(0), 0, b.data_ptr(), b.stride(0), 0, c.data_ptr(), g.data_ptr(),
         c.stride(0), M, N, K, _p(bias), _s())
    return c, g


def gemm_residual(a, b, res, *, bias=None, p: float = 0.0, seed: int = 0, stream_id: int = 0):
    """res + dropout_p(bf16(a @ b^T + bias)) in one GEMM (K-major operands)."""
    M, K = a.shape
    N = b.shape[0]
    c = torch.empty(M, N, device=a.device, dtype=torch.bfloat16)
    call("lynx_op_gemm_residual", a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0), M,
         N, K, _p(bias), res.data_ptr(), p, seed, stream_id, _s())
    return c


def gemm_gelu_bwd(a, b, x, *, b_mn: bool = False):
    """(a @ B^T) * gelu'(x) in one GEMM; B = b ([N,K]) or b.T (b_mn, b is [K,N])."""
    M, K = a.shape
    N = b.shape[1] if b_mn else b.shape[0]
    c = torch.empty(M, N, device=a.device, dtype=torch.bfloat16)
    call("lynx_op_gemm_gelu_bwd", a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), int(b_mn), c.data_ptr(),
         c.stride(0), M, N, K, x.data_ptr(), _s())
    return c


def layernorm_fwd(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float = 1e-5):
    rows, width = x.shape
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=x.device, dtype=torch.float32)
    rstd = torch.empty_like(mean)
    call("lynx_op_layernorm_fwd", x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(), mean.data_ptr(),
         rstd.data_ptr(), rows, width, eps, _s())
    return y, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd, dgamma_acc, dbeta_acc, dres=None):
    rows, width = x.shape
    dx = torch.empty_like(x)
    ws = torch.empty(lib().lynx_op_layernorm_bwd_workspace(rows, width) // 4 + 1, device=x.device,
                     dtype=torch.float32)
    call("lynx_op_layernorm_bwd", dy.data_ptr(), x.data_ptr(), gamma.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
         _p(dres), dx.data_ptr(), dgamma_acc.data_ptr(), dbeta_acc.data_ptr(), ws.data_ptr(), rows, width, _s())
    return dx


def bias_dropout_residual(y, bias, res, p: float, seed: int, stream_id: int):
    rows, width = y.shape
    out = torch.empty_like(y)
    call("lynx_op_bias_dropout_residual", y.data_ptr(), _p(bias), res.data_ptr(), out.data_ptr(), rows, width,
         float(p), seed, stream_id, _s())
    return out


def dropout_bwd(dout, p: float, seed: int, stream_id: int):
    rows, width = dout.shape
    dy = torch.empty_like(dout)
    call("lynx_op_dropout_bwd", dout.data_ptr(), dy.data_ptr(), rows, width, float(p), seed, stream_id, _s())
    return dy


def dropout_bwd_colsum(dout, acc, p: float, seed: int, stream_id: int):
    """(dropout_bwd(dout), acc += column sums of it) in one pass."""
    rows, width = dout.shape
    dy = torch.empty_like(dout)
    ws = torch.empty(lib().lynx_op_column_sum_workspace(rows, width) // 4 + 1, device=dout.device, dtype=torch.float32)
    call("lynx_op_dropout_bwd_colsum", dout.data_ptr(), dy.data_ptr(), acc.data_ptr(), ws.data_ptr(), rows, width,
         float(p), seed, stream_id, _s())
    return dy, acc


def column_sum_acc(x, acc):
    rows, width = x.shape
    if acc.numel() < width or not acc.is_contiguous():
        raise ValueError(f"column_sum_acc: accumulator of {acc.numel()} elements for width {width}")
    ws = torch.empty(lib().lynx_op_column_sum_workspace(rows, width) // 4 + 1, device=x.device, dtype=torch.float32)
    call("lynx_op_column_sum_acc", x.data_ptr(), acc.data_ptr(), ws.data_ptr(), rows, width, _s())
    return acc


def gelu_fwd(x):
    y = torch.empty_like(x)
    call("lynx_op_gelu_fwd", x.data_ptr(), y.data_ptr(), x.numel(), _s())
    return y


def gelu_bwd(dy, x):
    dx = torch.empty_like(x)
    call("lynx_op_gelu_bwd", dy.data_ptr(), x.data_ptr(), dx.data_ptr(), x.numel(), _s())
    return dx


def attention_fwd(qkv, batch: int, seq: int, heads: int, head_dim: int):
    out = torch.empty(batch * seq, heads * head_dim, device=qkv.device, dtype=torch.bfloat16)
    lse = torch.empty(batch, heads, seq, device=qkv.device, dtype=torch.float32)
    call("lynx_op_attention_fwd", qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), batch, seq, heads, head_dim, _s())
    return out, lse


def attention_bwd(qkv, out, dout, lse, batch: int, seq: int, heads: int, head_dim: int):
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(lib().lynx_op_attention_bwd_workspace(batch, seq, heads) // 4 + 1, device=qkv.device,
                     dtype=torch.float32)
    call("lynx_op_attention_bwd", qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dqkv.data_ptr(),
         ws.data_ptr(), batch, seq, heads, head_dim, _s())
    return dqkv


def embedding_fwd(tokens, wte, wpe, batch: int, seq: int, p: float, seed: int, stream_id: int):
    width = wte.shape[1]
    out = torch.empty(batch * seq, width, device=wte.device, dtype=torch.bfloat16)
    call("lynx_op_embedding_fwd", tokens.data_ptr(), wte.data_ptr(), wpe.data_ptr(), out.data_ptr(), batch, seq, width,
         float(p), seed, stream_id, _s())
    return out


def embedding_bwd(tokens, dout, dwte, dwpe, batch: int, seq: int, p: float, seed: int, stream_id: int):
    width = dwte.shape[1]
    ws = torch.empty(lib().lynx_op_embedding_bwd_workspace(batch, seq, width) // 4 + 1, device=dout.device,
                     dtype=torch.float32)
    call("lynx_op_embedding_bwd", tokens.data_ptr(), dout.data_ptr(), dwte.data_ptr(), dwpe.data_ptr(), ws.data_ptr(),
         batch, seq, width, dwte.shape[0], float(p), seed, stream_id, _s())


def xent_fwd_bwd(logits, labels, grad_scale: float):
    rows, vocab = logits.shape
    loss = torch.empty(rows, device=logits.device, dtype=torch.float32)
    call("lynx_op_xent_fwd_bwd", logits.data_ptr(), labels.data_ptr(), loss.data_ptr(), rows, vocab,
         float(grad_scale), _s())
    return loss


def adam(master, param, grad, m, v, *, lr, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0, step=1,
         grad_scale=1.0):
    call("lynx_op_adam", master.data_ptr(), param.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(),
         master.numel(), lr, beta1, beta2, eps, weight_decay, step, grad_scale, _s())


def init_normal(param, master, std: float, seed: int, stream_id: int):
    call("lynx_op_init_normal", param.data_ptr(), _p(master), param.numel(), std, seed, stream_id, _s())
