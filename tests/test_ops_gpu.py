"""Numerics of the sm_100a operator library against plain PyTorch fp32 references.

Tolerances (bf16 storage, fp32 accumulation): GEMM relative Frobenius error
<= 1e-2; elementwise / norm ops max |diff| <= 2 bf16 ulps of the output scale;
attention relative error <= 2e-2 (fwd) and <= 5e-2 (bwd). Determinism checks
(bit-identical reruns) back the recompute bit-identity requirement.
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / (b.norm() + 1e-12)).item()


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2406_08756_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 384, 192), (512, 1536, 512), (1024, 2048, 1024)])
def test_gemm_majors(ops, cuda, a_mn, b_mn, M, N, K):
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    a = A.t().contiguous() if a_mn else A
    b = B.t().contiguous() if b_mn else B
    ref = A.float() @ B.float().t()
    out = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    assert rel(out, ref) < 1e-2


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("mode", [1, 0, 2])
def test_gemm_pair_and_single_cta(ops, cuda, a_mn, b_mn, mode):
    """512x256 "wide" CTA-pair tiles (mode 2), 256x256 CTA-pair (cta_group::2) tiles (mode 1) and the
    128xBN single-CTA kernel (mode 0) on shapes all accept; bf16+bias (TMA-store) and fp32-accumulate epilogues."""
    from paper_2406_08756_b200._native import lib
    M, N, K = (4096, 2048, 640) if mode == 2 else (2048, 1536, 640)
    g = torch.Generator(device=cuda).manual_seed(11)
    A = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    B = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    a = A.t().contiguous() if a_mn else A
    b = B.t().contiguous() if b_mn else B
    bias = torch.randn(N, device=cuda, generator=g).bfloat16()
    lib().lynx_op_gemm_mode(mode)
    try:
        out = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, bias=bias)
        acc = torch.ones(M, N, device=cuda)
        ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, out=acc, epi=ops.EPI_ACC_F32)
        torch.cuda.synchronize()
    finally:
        lib().lynx_op_gemm_mode(-1)
    ref = A.float() @ B.float().t()
    assert rel(out, ref + bias.float()) < 1e-2
    assert rel(acc, ref + 1) < 1e-5


@pytest.mark.parametrize("mode,M,N,K", [(-1, 512, 1024, 256), (0, 256, 384, 128), (1, 512, 512, 192),
                                        (2, 1024, 2048, 8192)])
def test_gemm_gelu_epilogue_matches_gelu_kernel(ops, cuda, mode, M, N, K):
    """The fused FC1+GeLU epilogue writes C and gelu(C); gelu(C) must equal the stand-alone GeLU
    kernel on C bit for bit (a recomputed GeLU may come from either path)."""
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    a = (torch.randn(M, K, device=cuda, generator=g) * 0.3).bfloat16()
    b = (torch.randn(N, K, device=cuda, generator=g) * 0.3).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g).bfloat16()
    lib().lynx_op_gemm_mode(mode)
    try:
        c, gc = ops.gemm_gelu(a, b, bias=bias)
        c_ref = ops.gemm(a, b, bias=bias)
    finally:
        lib().lynx_op_gemm_mode(-1)
    assert torch.equal(c, c_ref)
    assert torch.equal(gc, ops.gelu_fwd(c))


@pytest.mark.parametrize("mode,M,N,K,p", [(-1, 512, 1024, 256, 0.1), (0, 256, 384, 128, 0.1), (-1, 1024, 2048, 8192, 0.0),
                                          (1, 512, 512, 192, 0.5)])
def test_gemm_residual_epilogue(ops, cuda, mode, M, N, K, p):
    """Projection + bias + dropout + residual fused in the GEMM epilogue: the same keep mask as the
    two-kernel path (GEMM, then bias_dropout_residual), values within one bf16 rounding; reruns
    are bit-identical (a regenerated PROJ_RES / FC2_RES must equal the forward's)."""
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N + K)
    a = (torch.randn(M, K, device=cuda, generator=g) * 0.3).bfloat16()
    b = (torch.randn(N, K, device=cuda, generator=g) * 0.3).bfloat16()
    bias = torch.randn(N, device=cuda, generator=g).bfloat16()
    res = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    lib().lynx_op_gemm_mode(mode)
    try:
        out = ops.gemm_residual(a, b, res, bias=bias, p=p, seed=7, stream_id=11)
        out2 = ops.gemm_residual(a, b, res, bias=bias, p=p, seed=7, stream_id=11)
        y = ops.gemm(a, b, bias=bias)
    finally:
        lib().lynx_op_gemm_mode(-1)
    ref = ops.bias_dropout_residual(y, None, res, p, 7, 11)
    assert torch.equal(out, out2)
    kept_fused = out != res
    kept_ref = ref != res
    assert (kept_fused == kept_ref).float().mean() > 0.999  # same mask (ties where y*scale rounds to 0)
    assert rel(out, ref) < 1e-2


@pytest.mark.parametrize("mode,M,N,K", [(-1, 512, 1024, 256), (0, 256, 384, 128), (1, 512, 2048, 512)])
def test_gemm_gelu_bwd_epilogue(ops, cuda, mode, M, N, K):
    """GeLU backward fused into the dX GEMM (B MN-major, as the executor calls it) vs GEMM + gelu_bwd."""
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(M + 3 * N + K)
    a = (torch.randn(M, K, device=cuda, generator=g) * 0.3).bfloat16()
    bt = (torch.randn(K, N, device=cuda, generator=g) * 0.3).bfloat16()  # stored [K][N]
    x = torch.randn(M, N, device=cuda, generator=g).bfloat16()
    lib().lynx_op_gemm_mode(mode)
    try:
        fused = ops.gemm_gelu_bwd(a, bt, x, b_mn=True)
        dg = ops.gemm(a, bt, b_mn=True)
    finally:
        lib().lynx_op_gemm_mode(-1)
    ref = ops.gelu_bwd(dg, x)
    assert rel(fused, ref) < 1e-2


@pytest.mark.parametrize("mode", [1, 2, -1])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (True, True), (False, True)])
def test_gemm_pair_edge_tiles(ops, cuda, mode, a_mn, b_mn):
    """CTA-pair kernels on 128-aligned shapes that are not tile multiples (M = 2.5 x 256 rows of the
    pair tile, N = 4.5 x 256: the LM head's V = 50304 case): TMA zero-fills the loads, the TMA store
    clips and the direct epilogues bounds-check."""
    from paper_2406_08756_b200._native import lib
    M, N, K = 5 * 128 * (2 if mode == 2 else 1), 9 * 128, 512
    g = torch.Generator(device=cuda).manual_seed(M + N)
    A = (torch.randn(M, K, device=cuda, generator=g) * 0.3).bfloat16()
    B = (torch.randn(N, K, device=cuda, generator=g) * 0.3).bfloat16()
    a = A.t().contiguous() if a_mn else A
    b = B.t().contiguous() if b_mn else B
    bias = torch.randn(N, device=cuda, generator=g).bfloat16()
    ref = A.float() @ B.float().t()
    lib().lynx_op_gemm_mode(mode)
    try:
        out = ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, bias=bias)
        acc = torch.ones(M, N, device=cuda)
        ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, out=acc, epi=ops.EPI_ACC_F32)
        accb = torch.ones(M, N, device=cuda, dtype=torch.bfloat16)
        ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, out=accb, epi=ops.EPI_ACC_BF16)
        torch.cuda.synchronize()
    finally:
        lib().lynx_op_gemm_mode(-1)
    assert rel(out, ref + bias.float()) < 1e-2
    assert rel(acc, ref + 1) < 1e-5
    assert rel(accb, ref + 1) < 1e-2


def test_gemm_bias_and_f32_epilogues(ops, cuda):
    g = torch.Generator(device=cuda).manual_seed(7)
    A = torch.randn(256, 512, device=cuda, generator=g).bfloat16()
    B = torch.randn(768, 512, device=cuda, generator=g).bfloat16()
    bias = torch.randn(768, device=cuda, generator=g).bfloat16()
    ref = A.float() @ B.float().t()
    out = ops.gemm(A, B, bias=bias)
    assert rel(out, ref + bias.float()) < 1e-2
    acc = torch.ones(256, 768, device=cuda)
    ops.gemm(A, B, out=acc, epi=ops.EPI_ACC_F32)
    assert rel(acc, ref + 1) < 1e-5
    f = ops.gemm(A, B, epi=ops.EPI_F32)
    assert rel(f, ref) < 1e-5


def test_gemm_deterministic(ops, cuda):
    A = torch.randn(1024, 1024, device=cuda).bfloat16()
    B = torch.randn(1024, 1024, device=cuda).bfloat16()
    o1 = ops.gemm(A, B)
    o2 = ops.gemm(A, B)
    assert torch.equal(o1, o2)


def test_gemm_rejects_bad_shapes(ops, cuda):
    from paper_2406_08756_b200._native import LynxError
    A = torch.randn(100, 64, device=cuda).bfloat16()
    with pytest.raises(LynxError):
        ops.gemm(A, A)


@pytest.mark.parametrize("rows,width", [(64, 512), (300, 1792), (128, 4096), (17, 6144), (1000, 4096), (2001, 5120),
                                        (50, 1000)])
def test_layernorm(ops, cuda, rows, width):
    x = torch.randn(rows, width, device=cuda).bfloat16()
    gam = (1 + 0.1 * torch.randn(width, device=cuda)).bfloat16()
    bet = (0.1 * torch.randn(width, device=cuda)).bfloat16()
    y, mean, rstd = ops.layernorm_fwd(x, gam, bet)
    xr = x.float().requires_grad_()
    gr = gam.float().requires_grad_()
    br = bet.float().requires_grad_()
    yr = torch.nn.functional.layer_norm(xr, (width,), gr, br, eps=1e-5)
    assert (y.float() - yr).abs().max().item() < 3e-2
    assert torch.allclose(mean, x.float().mean(1), atol=1e-4)
    dy = torch.randn(rows, width, device=cuda).bfloat16()
    dres = torch.randn(rows, width, device=cuda).bfloat16()
    yr.backward(dy.float())
    dg = torch.zeros(width, device=cuda)
    db = torch.zeros(width, device=cuda)
    dx = ops.layernorm_bwd(dy, x, gam, mean, rstd, dg, db, dres=dres)
    assert rel(dx, xr.grad + dres.float()) < 1e-2
    assert rel(dg, gr.grad) < 1e-3
    assert rel(db, br.grad) < 1e-3
    dg2 = torch.zeros(width, device=cuda)
    db2 = torch.zeros(width, device=cuda)
    dx2 = ops.layernorm_bwd(dy, x, gam, mean, rstd, dg2, db2, dres=dres)
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2) and torch.equal(db, db2)


def test_dropout_residual_replays_mask(ops, cuda):
    rows, width = 512, 1024
    y = torch.randn(rows, width, device=cuda).bfloat16()
    b = torch.randn(width, device=cuda).bfloat16()
    r = torch.randn(rows, width, device=cuda).bfloat16()
    o1 = ops.bias_dropout_residual(y, b, r, 0.1, seed=42, stream_id=1234)
    o2 = ops.bias_dropout_residual(y, b, r, 0.1, seed=42, stream_id=1234)
    o3 = ops.bias_dropout_residual(y, b, r, 0.1, seed=42, stream_id=1235)
    assert torch.equal(o1, o2)
    assert not torch.equal(o1, o3)
    ones = torch.ones_like(y)
    keep = ops.bias_dropout_residual(ones, None, torch.zeros_like(y), 0.1, seed=42, stream_id=1234).float() != 0
    frac = keep.float().mean().item()
    assert abs(frac - 0.9) < 0.01
    ref = r.float() + keep.float() * (y.float() + b.float()) / 0.9
    assert (o1.float() - ref).abs().max().item() < 0.05
    o0 = ops.bias_dropout_residual(y, b, r, 0.0, seed=42, stream_id=1)
    assert (o0.float() - (r.float() + y.float() + b.float())).abs().max().item() < 0.05
    dout = torch.randn(rows, width, device=cuda).bfloat16()
    dy = ops.dropout_bwd(dout, 0.1, seed=42, stream_id=1234)
    assert (dy.float() - keep.float() * dout.float() / 0.9).abs().max().item() < 0.02


def test_column_sum(ops, cuda):
    x = torch.randn(5000, 768, device=cuda).bfloat16()
    acc = torch.full((768,), 2.0, device=cuda)
    ops.column_sum_acc(x, acc)
    assert torch.allclose(acc, x.float().sum(0) + 2, atol=1e-2)


@pytest.mark.parametrize("rows,width,p", [(65536 // 8, 4096, 0.1), (5000, 768, 0.1), (777, 1024, 0.0)])
def test_dropout_bwd_colsum_matches_two_kernels(ops, cuda, rows, width, p):
    """The fused branch-gradient + bias-gradient pass equals dropout_bwd then column_sum_acc bit for bit."""
    dout = torch.randn(rows, width, device=cuda).bfloat16()
    acc1 = torch.full((width,), 0.5, device=cuda)
    acc2 = acc1.clone()
    dy1 = ops.dropout_bwd(dout, p, seed=7, stream_id=99)
    ops.column_sum_acc(dy1, acc1)
    dy2, _ = ops.dropout_bwd_colsum(dout, acc2, p, seed=7, stream_id=99)
    assert torch.equal(dy1, dy2)
    assert torch.equal(acc1, acc2)


def test_gelu(ops, cuda):
    x = (3 * torch.randn(4096, 256, device=cuda)).bfloat16()
    y = ops.gelu_fwd(x)
    xr = x.float().requires_grad_()
    yr = torch.nn.functional.gelu(xr, approximate="tanh")
    assert (y.float() - yr).abs().max().item() < 3e-2
    dy = torch.randn_like(x)
    yr.backward(dy.float())
    dx = ops.gelu_bwd(dy, x)
    assert rel(dx, xr.grad) < 1e-2


def _ref_attention(qkv, B, S, H, D):
    q, k, v = qkv.float().view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    att = (q @ k.transpose(-1, -2)) / math.sqrt(D)
    mask = torch.ones(S, S, device=qkv.device, dtype=torch.bool).triu(1)
    att = att.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(att, -1)
    o = torch.softmax(att, -1) @ v
    return o.permute(0, 2, 1, 3).reshape(B * S, H * D), lse


@pytest.mark.parametrize("mode", [-1, 0])
@pytest.mark.parametrize("B,S,H,D", [(2, 128, 2, 64), (1, 256, 3, 128), (2, 192, 2, 96), (1, 128, 2, 112),
                                     (2, 640, 2, 128), (1, 1024, 1, 64), (1, 256, 4, 64), (2, 256, 3, 96),
                                     (1, 384, 2, 112), (1, 2048, 2, 96), (1, 2048, 2, 112)])
def test_attention(ops, cuda, B, S, H, D, mode):
    """mode -1: tcgen05 kernels where the shape allows (D 64/96/112/128, S % 128 == 0); 0: mma.sync kernels."""
    from paper_2406_08756_b200._native import lib
    assert lib().lynx_op_attention_tc_supported(S, D) == (1 if S % 128 == 0 else 0)
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(B * S * H * D)
    qkv = torch.randn(B * S, 3 * H * D, device=cuda, generator=g).bfloat16()
    lib().lynx_op_attention_mode(mode)
    try:
        _check_attention(ops, cuda, qkv, g, B, S, H, D)
    finally:
        lib().lynx_op_attention_mode(-1)


def _check_attention(ops, cuda, qkv, g, B, S, H, D):
    out, lse = ops.attention_fwd(qkv, B, S, H, D)
    x = qkv.float().requires_grad_()
    ref, ref_lse = _ref_attention(x, B, S, H, D)
    assert rel(out, ref) < 2e-2
    assert torch.allclose(lse, ref_lse, atol=2e-3)
    dout = torch.randn(B * S, H * D, device=cuda, generator=g).bfloat16()
    ref.backward(dout.float())
    dqkv = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
    assert rel(dqkv, x.grad) < 5e-2
    dqkv2 = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
    assert torch.equal(dqkv, dqkv2)


@pytest.mark.parametrize("B,S,H,D", [(2, 512, 3, 128), (1, 1024, 2, 64), (2, 384, 2, 112), (1, 256, 2, 96)])
def test_attention_bwd_warpgroup_variants_are_bit_identical(ops, cuda, B, S, H, D):
    """The tcgen05 backward kernels with 2 or 4 row warpgroups (64 / kWG columns each) issue the same MMAs
    in the same order on the same per-element values: dQ, dK, dV are bit-identical."""
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(S + D)
    qkv = torch.randn(B * S, 3 * H * D, device=cuda, generator=g).bfloat16()
    dout = torch.randn(B * S, H * D, device=cuda, generator=g).bfloat16()
    out, lse = ops.attention_fwd(qkv, B, S, H, D)
    res = {}
    try:
        for wg in (2, 4):
            lib().lynx_op_attention_bwd_warpgroups(wg)
            res[wg] = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
    finally:
        lib().lynx_op_attention_bwd_warpgroups(0)
    torch.cuda.synchronize()
    assert torch.equal(res[2], res[4])


@pytest.mark.parametrize("B,S,H,D", [(2, 512, 3, 128), (1, 384, 2, 64), (2, 640, 2, 112), (1, 128, 2, 96),
                                     (1, 2048, 2, 128)])
def test_attention_fwd_two_tile_kernel_is_bit_identical(ops, cuda, B, S, H, D):
    """The two-query-tile forward (two softmax warpgroups ping-ponging on the tensor core) computes every row
    exactly as the one-tile kernel: O and lse are bit-identical, odd tile counts included."""
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(S * D + H)
    qkv = torch.randn(B * S, 3 * H * D, device=cuda, generator=g).bfloat16()
    res = {}
    try:
        for tiles in (1, 2):
            lib().lynx_op_attention_fwd_tiles(tiles)
            res[tiles] = ops.attention_fwd(qkv, B, S, H, D)
    finally:
        lib().lynx_op_attention_fwd_tiles(0)
    torch.cuda.synchronize()
    assert torch.equal(res[1][0], res[2][0]) and torch.equal(res[1][1], res[2][1])


@pytest.mark.parametrize("tiles", [1, 3, 4])
@pytest.mark.parametrize("B,S,H,D", [(2, 512, 3, 128), (1, 384, 2, 64), (2, 640, 2, 112), (1, 128, 2, 96),
                                     (1, 2048, 2, 128), (1, 2048, 2, 96), (3, 256, 1, 64)])
def test_attention_fwd_variants_match_reference(ops, cuda, B, S, H, D, tiles):
    """The one-tile, the 64-key-block (attn_fwd3_tc_kernel: separate P region, one MMA issuer per query
    tile) and the CTA-pair forward (attn_fwd4_tc_kernel, D = 128 with an even tile count; other shapes run
    the two-tile kernel) against fp32 PyTorch, forward and backward (the backward consumes their lse), odd
    tile counts included; reruns are bit-identical."""
    from paper_2406_08756_b200._native import lib
    g = torch.Generator(device=cuda).manual_seed(S * D + H + tiles)
    qkv = torch.randn(B * S, 3 * H * D, device=cuda, generator=g).bfloat16()
    try:
        lib().lynx_op_attention_fwd_tiles(tiles)
        _check_attention(ops, cuda, qkv, g, B, S, H, D)
        a, b = ops.attention_fwd(qkv, B, S, H, D), ops.attention_fwd(qkv, B, S, H, D)
    finally:
        lib().lynx_op_attention_fwd_tiles(0)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_xent(ops, cuda):
    rows, V = 256, 1024
    logits = torch.randn(rows, V, device=cuda).bfloat16()
    labels = torch.randint(0, V, (rows,), device=cuda, dtype=torch.int32)
    x = logits.float().requires_grad_()
    ref = torch.nn.functional.cross_entropy(x, labels.long(), reduction="none")
    ref.sum().backward()
    work = logits.clone()
    loss = ops.xent_fwd_bwd(work, labels, 1.0)
    assert torch.allclose(loss, ref, atol=2e-3)
    assert (work.float() - x.grad).abs().max().item() < 1e-2


def test_embedding(ops, cuda):
    B, S, W, V = 2, 64, 256, 512
    tok = torch.randint(0, V, (B * S,), device=cuda, dtype=torch.int32)
    wte = torch.randn(V, W, device=cuda).bfloat16()
    wpe = torch.randn(S, W, device=cuda).bfloat16()
    out = ops.embedding_fwd(tok, wte, wpe, B, S, 0.0, 1, 2)
    ref = wte.float()[tok.long()] + wpe.float().repeat(B, 1)
    assert (out.float() - ref).abs().max().item() < 3e-2
    dout = torch.randn(B * S, W, device=cuda).bfloat16()
    dwte = torch.zeros(V, W, device=cuda)
    dwpe = torch.zeros(S, W, device=cuda)
    ops.embedding_bwd(tok, dout, dwte, dwpe, B, S, 0.0, 1, 2)
    ref_wte = torch.zeros(V, W, device=cuda).index_add_(0, tok.long(), dout.float())
    assert torch.allclose(dwte, ref_wte, atol=1e-3)
    assert torch.allclose(dwpe, dout.float().view(B, S, W).sum(0), atol=1e-3)


@pytest.mark.parametrize("B,S,W,V,p", [(2, 64, 256, 512, 0.0), (2, 64, 256, 512, 0.1), (1, 300, 64, 7, 0.0),
                                       (4, 2048, 512, 512, 0.1)])
def test_embedding_bwd_deterministic_under_collisions(ops, cuda, B, S, W, V, p):
    """Sorted segment sums (no atomics): bit-identical reruns even when every token repeats many times
    (V = 7 / 512 over up to 8192 positions), equal to a float64 index_add with the executor's Philox mask."""
    import numpy as np
    from oracle import gpt_oracle
    g = torch.Generator(device=cuda).manual_seed(B * S + V)
    tok = torch.randint(0, V, (B * S,), device=cuda, dtype=torch.int32, generator=g)
    dout = torch.randn(B * S, W, device=cuda, generator=g).bfloat16()
    runs = []
    for _ in range(3):
        dwte = torch.zeros(V, W, device=cuda)
        dwpe = torch.zeros(S, W, device=cuda)
        ops.embedding_bwd(tok, dout, dwte, dwpe, B, S, p, 77, 5)
        runs.append((dwte.cpu(), dwpe.cpu()))
    for a, b in runs[1:]:
        assert torch.equal(a, runs[0][0]) and torch.equal(b, runs[0][1])
    keep = torch.from_numpy(gpt_oracle.keep_mask(77, 5, B * S * W, p).reshape(B * S, W))
    scale = float(np.float32(1) / (np.float32(1) - np.float32(p))) if p > 0 else 1.0
    d = torch.where(keep, dout.cpu().double() * scale, torch.zeros((), dtype=torch.float64))
    ref_wte = torch.zeros(V, W, dtype=torch.float64).index_add_(0, tok.cpu().long(), d)
    ref_wpe = d.view(B, S, W).sum(0)
    assert (runs[0][0].double() - ref_wte).abs().max().item() < 1e-4 * max(1.0, ref_wte.abs().max().item())
    assert (runs[0][1].double() - ref_wpe).abs().max().item() < 1e-4 * max(1.0, ref_wpe.abs().max().item())


def test_dropout_mask_matches_oracle_philox(ops, cuda):
    """The device Philox-4x32-10 dropout mask equals the oracle's numpy restatement element for element."""
    from oracle import gpt_oracle
    rows, width, p = 64, 1024, 0.1
    ones = torch.ones(rows, width, device=cuda, dtype=torch.bfloat16)
    out = ops.dropout_bwd(ones, p, 1000045, (3 << 32) | (1 << 8) | 5)
    keep = gpt_oracle.keep_mask(1000045, (3 << 32) | (1 << 8) | 5, rows * width, p)
    assert torch.equal(out.cpu().flatten() != 0, torch.from_numpy(keep))


def test_adam_and_init(ops, cuda):
    n = 10000
    p = torch.empty(n, device=cuda, dtype=torch.bfloat16)
    master = torch.empty(n, device=cuda)
    ops.init_normal(p, master, 0.02, seed=42, stream_id=3)
    assert abs(master.std().item() - 0.02) < 2e-3
    assert torch.equal(master, p.float())
    g = torch.randn(n, device=cuda)
    m = torch.zeros(n, device=cuda)
    v = torch.zeros(n, device=cuda)
    ref = master.clone().requires_grad_()
    opt = torch.optim.AdamW([ref], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    ref.grad = g.clone()
    opt.step()
    ops.adam(master, p, g, m, v, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, step=1)
    assert torch.allclose(master, ref.detach(), atol=1e-6)
