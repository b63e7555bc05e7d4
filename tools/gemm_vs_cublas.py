"""One FC1-forward GEMM [T,16384,4096] through this repo's tcgen05 kernel, then through cuBLAS
(torch.matmul), for side-by-side ncu captures:
    ncu --set full -k regex:'gemm2|nvjet|sm100|cutlass' -c 2 python tools/gemm_vs_cublas.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
h = 4096
x = torch.randn(T, h, device="cuda").bfloat16()
w = torch.randn(4 * h, h, device="cuda").bfloat16()
y = torch.empty(T, 4 * h, device="cuda", dtype=torch.bfloat16)
ops.gemm(x, w, out=y)
torch.cuda.synchronize()
torch.matmul(x, w.t(), out=y)
torch.cuda.synchronize()
print("ok")
