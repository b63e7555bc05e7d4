"""Run the bench's dominant GEMM shapes a few times (target for ncu --set full captures).

    python tools/gemm_one.py [T]   -> 4x FC1 forward with the fused GeLU epilogue [T,16384,4096] (as in the
                                      training step), then 4x FC1 dW [16384,4096,T] (bf16 store epilogue),
                                      then 4x FC2 dX with the fused GeLU backward [T,16384,4096] (FC1 output
                                      read by TMA in the epilogue)
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
w2 = torch.randn(h, 4 * h, device="cuda").bfloat16()  # W_fc2 [h, 4h], read MN-major as B
for _ in range(4):
    ops.gemm_gelu_bwd(x, w2, y, b_mn=True)
torch.cuda.synchronize()
print("ok")
