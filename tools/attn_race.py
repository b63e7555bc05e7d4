"""Hunt a rare run-to-run difference in the tcgen05 attention backward: many repetitions with the
allocator perturbed between calls; reports how often and where (Q / K / V part, rows) results differ.

    python tools/attn_race.py [reps] [B S H D]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    B, S, H, D = (int(x) for x in sys.argv[2:6]) if len(sys.argv) > 5 else (1, 1024, 1, 64)
    g = torch.Generator(device="cuda").manual_seed(B * S * H * D)
    qkv = torch.randn(B * S, 3 * H * D, device="cuda", generator=g).bfloat16()
    out, lse = ops.attention_fwd(qkv, B, S, H, D)
    dout = torch.randn(B * S, H * D, device="cuda", generator=g).bfloat16()
    ref = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
    nbad, where = 0, {}
    junk = []
    for i in range(reps):
        junk.append(torch.empty(int(torch.randint(1, 1 << 20, (1,))), device="cuda"))
        if len(junk) > 8:
            junk.pop(0)
        if i % 3 == 0:
            out2, lse2 = ops.attention_fwd(qkv, B, S, H, D)
            if not (torch.equal(out2, out) and torch.equal(lse2, lse)):
                where["fwd"] = where.get("fwd", 0) + 1
        d = ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
        if not torch.equal(d, ref):
            nbad += 1
            diff = (d.float() - ref.float()).abs().view(B, S, 3, H, D)
            for j, n in enumerate("qkv"):
                if diff[:, :, j].max() > 0:
                    rows = torch.nonzero(diff[:, :, j].amax(dim=(2, 3)))[:, 1]
                    key = f"{n}: rows {rows.min().item()}-{rows.max().item()} ({rows.numel()}), max {diff[:, :, j].max().item():.3g}"
                    where[key] = where.get(key, 0) + 1
    print(f"B{B} S{S} H{H} D{D}: {nbad}/{reps} backward runs differ; {where}", flush=True)


if __name__ == "__main__":
    main()
