"""Run the bench's dominant GEMM shapes a few times (target for ncu --set full captures).

    python tools/gemm_one.py [T]   -> 4x FC1 forward with the fused GeLU epilogue [T,16384,4096] (as in the
                                      training step), then 4x FC1 dW [16384,4096,T] (bf16 store epilogue)
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
h = 4096
x = torch.randn(T, h, device="cuda").bfloat16()
w = torch.randn(4 * h, h, device="cuda").bfloat16()
b = torch.randn(4 * h, device="cuda").bfloat16()
for _ in range(4):
    y, g = ops.gemm_gelu(x, w, bias=b)
gw = torch.empty(4 * h, h, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    ops.gemm(y, x, a_mn=True, b_mn=True, out=gw, epi=ops.EPI_BF16)
torch.cuda.synchronize()
print("ok")
