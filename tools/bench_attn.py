"""Time the attention kernels (tcgen05 vs mma.sync) on the GPT-7B per-layer shape.

    python tools/bench_attn.py [B S H D]
Prints ms and causal TFLOP/s (fwd 2 matmuls, bwd 5 matmuls over the causal half).
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402
from paper_2406_08756_b200._native import lib  # noqa: E402


def timeit(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    B, S, H, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (16, 2048, 32, 128)
    qkv = (torch.randn(B * S, 3 * H * D, device="cuda") * 0.5).bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    f_fwd = 4.0 * B * H * S * S * D / 2
    res = {}
    for mode in (0, -1):
        lib().lynx_op_attention_mode(mode)
        out, lse = ops.attention_fwd(qkv, B, S, H, D)
        tf = timeit(lambda: ops.attention_fwd(qkv, B, S, H, D))
        tb = timeit(lambda: ops.attention_bwd(qkv, out, dout, lse, B, S, H, D))
        d = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
        res[mode] = (out.float(), d.float())
        print(f"mode {mode:2d}: fwd {tf:7.3f} ms {f_fwd / tf / 1e9:7.1f} TF/s | bwd {tb:7.3f} ms "
              f"{2.5 * f_fwd / tb / 1e9:7.1f} TF/s", flush=True)
    lib().lynx_op_attention_mode(-1)
    out, lse = ops.attention_fwd(qkv, B, S, H, D)
    for wg in (2, 4):  # row warpgroups of the tcgen05 backward kernels
        lib().lynx_op_attention_bwd_warpgroups(wg)
        tb = timeit(lambda: ops.attention_bwd(qkv, out, dout, lse, B, S, H, D))
        print(f"tcgen05 bwd, {wg} row warpgroups: {tb:7.3f} ms {2.5 * f_fwd / tb / 1e9:7.1f} TF/s", flush=True)
    lib().lynx_op_attention_bwd_warpgroups(0)
    for tiles in (1, 2, 3, 4):  # tcgen05 forward variant (3: 64-key blocks, P apart from S; 4: CTA pair)
        lib().lynx_op_attention_fwd_tiles(tiles)
        tf = timeit(lambda: ops.attention_fwd(qkv, B, S, H, D))
        print(f"tcgen05 fwd, {tiles} query tile(s) per CTA: {tf:7.3f} ms {f_fwd / tf / 1e9:7.1f} TF/s", flush=True)
    lib().lynx_op_attention_fwd_tiles(0)
    for i, name in enumerate(["out", "dqkv"]):
        a, b = res[-1][i], res[0][i]
        print(name, "rel diff tc vs mma:", ((a - b).norm() / b.norm()).item())


if __name__ == "__main__":
    main()
