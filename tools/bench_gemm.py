"""Micro-benchmark of the tcgen05 GEMM at the GPT-7B per-rank shapes (CUDA events, L2-sized inputs).

cuBLAS (torch.matmul) is timed beside it as a yardstick only.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    h = 4096
    shapes = [("qkv_fwd", T, 3 * h, h, False, False), ("fc1_fwd", T, 4 * h, h, False, False),
              ("fc2_fwd", T, h, 4 * h, False, False), ("fc1_dx", T, h, 4 * h, False, True),
              ("fc1_dw", 4 * h, h, T, True, True), ("proj_dw", h, h, T, True, True)]
    modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [-1]
    from paper_2406_08756_b200._native import lib
    res = []
    for name, M, N, K, amn, bmn in shapes:
        a = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
        b = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
        epis = [ops.EPI_ACC_F32, ops.EPI_F32] if name.endswith("dw") else [ops.EPI_BF16]
        A = a.t() if amn else a
        B = b if bmn else b.t()
        ms_cb = timeit(lambda: torch.matmul(A, B))
        fl = 2.0 * M * N * K
        for mode in modes:
            lib().lynx_op_gemm_mode(mode)
            for epi in epis:
                out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi else torch.bfloat16)
                ms = timeit(lambda: ops.gemm(a, b, a_mn=amn, b_mn=bmn, out=out, epi=epi))
                res.append({"gemm": name, "mode": mode, "epi": epi, "M": M, "N": N, "K": K, "ms": round(ms, 4),
                            "tflops": round(fl / ms / 1e9, 1), "cublas_tflops": round(fl / ms_cb / 1e9, 1)})
                print(json.dumps(res[-1]), flush=True)
                del out
        lib().lynx_op_gemm_mode(-1)


if __name__ == "__main__":
    main()
