"""Repeat the tcgen05 attention backward on fixed inputs and report run-to-run differences
(dQ / dK / dV regions separately): a race shows up as occasional mismatches.

    python tools/attn_determinism.py [reps]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402


def bwd_into(qkv, out, dout, lse, B, S, H, D, fill, ws_fill):
    """attention_bwd into a pre-filled output and workspace: entries the kernels never write keep `fill`."""
    from paper_2406_08756_b200._native import lib
    dqkv = torch.full_like(qkv, fill)
    ws = torch.full((lib().lynx_op_attention_bwd_workspace(B, S, H) // 4 + 1,), ws_fill, device=qkv.device)
    ops.call("lynx_op_attention_bwd", qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
             dqkv.data_ptr(), ws.data_ptr(), B, S, H, D, ops._s())
    return dqkv


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    for (B, S, H, D) in [(1, 1024, 1, 64), (1, 256, 4, 64), (2, 640, 2, 128), (4, 2048, 8, 128), (1, 1024, 2, 128)]:
        g = torch.Generator(device="cuda").manual_seed(B * S * H * D)
        qkv = torch.randn(B * S, 3 * H * D, device="cuda", generator=g).bfloat16()
        out, lse = ops.attention_fwd(qkv, B, S, H, D)
        outs = [ops.attention_fwd(qkv, B, S, H, D)[0] for _ in range(5)]
        fwd_bad = sum(int(not torch.equal(o, out)) for o in outs)
        dout = torch.randn(B * S, H * D, device="cuda", generator=g).bfloat16()
        ref = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
        bad = {"q": 0, "k": 0, "v": 0}
        worst = 0.0
        for _ in range(reps):
            d = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
            diff = (d.float() - ref.float()).abs().view(B * S, 3, H * D)
            for i, n in enumerate("qkv"):
                if diff[:, i].max().item() > 0:
                    bad[n] += 1
            worst = max(worst, diff.max().item())
        a = bwd_into(qkv, out, dout, lse, B, S, H, D, float("nan"), 0.0)
        b = bwd_into(qkv, out, dout, lse, B, S, H, D, 0.0, float("nan"))
        unwritten = int(torch.isnan(a.float()).sum().item())
        ws_dep = int((torch.isnan(b.float()) | (b != ref)).sum().item())
        print(f"   unwritten dqkv entries {unwritten}, entries that depend on workspace contents {ws_dep}, "
              f"differ from ref with zeroed out {int((bwd_into(qkv, out, dout, lse, B, S, H, D, 0.0, 0.0) != ref).sum())}")
        rows = None
        if worst > 0:
            diff = (d.float() - ref.float()).abs().view(B * S, 3, H * D).amax(dim=(1, 2))
            rows = torch.nonzero(diff).flatten()[:10].tolist()
        print(f"B{B} S{S} H{H} D{D}: fwd mismatches {fwd_bad}/5, bwd mismatching runs per region {bad} of {reps}, "
              f"max |diff| {worst:.4g}, rows {rows}", flush=True)


if __name__ == "__main__":
    main()
