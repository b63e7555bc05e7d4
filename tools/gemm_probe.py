"""GEMM kernel variants on one shape: single-CTA vs CTA-pair; full / no epilogue (99) / MMA only (98) /
pair with per-CTA TMA signalling only the CTA's own barrier (97, K-major only, timing only).

    python tools/gemm_probe.py [T]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402
from paper_2406_08756_b200._native import lib  # noqa: E402


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
h = 4096
for (name, M, N, K, amn, bmn, epi) in [("fc1_fwd", T, 4 * h, h, False, False, 0),
                                       ("fc1_dw", 4 * h, h, T, True, True, 1)]:
    a = torch.randn(K, M, device="cuda").bfloat16() if amn else torch.randn(M, K, device="cuda").bfloat16()
    b = torch.randn(K, N, device="cuda").bfloat16() if bmn else torch.randn(N, K, device="cuda").bfloat16()
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi else torch.bfloat16)
    for mode in (0, 1):
        lib().lynx_op_gemm_mode(mode)
        variants = (epi, 99, 98) + ((97,) if (mode == 1 and not amn and not bmn) else ())
        for e in variants:
            ms = timeit(lambda: ops.gemm(a, b, a_mn=amn, b_mn=bmn, out=out, epi=e))
            print(json.dumps({"gemm": name, "mode": "pair" if mode else "single",
                              "variant": {97: "own-barrier-tma", 98: "mma-only", 99: "no-epilogue"}.get(e, f"epi{e}"),
                              "ms": round(ms, 4), "tflops": round(2.0 * M * N * K / ms / 1e9, 1)}), flush=True)
    lib().lynx_op_gemm_mode(-1)
