"""Wave quantization of the weight-gradient GEMMs at the GPT-7B shapes (T = 65536, h = 4096): time per
launch and TFLOP/s of each dW shape with the wide (512 x 256) and the 256 x 256 CTA-pair tiles.

    python tools/gemm_waves.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402
from paper_2406_08756_b200._native import lib  # noqa: E402


def timeit(fn, iters=10):
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
    T, h = 65536, 4096
    x = torch.randn(T, h, device="cuda").bfloat16()
    for name, m in (("qkv dW", 3 * h), ("proj dW", h), ("fc1 dW", 4 * h)):
        dy = torch.randn(T, m, device="cuda").bfloat16()
        fl = 2.0 * T * m * h
        for mode, label in ((2, "wide 512x256"), (1, "pair 256x256")):
            lib().lynx_op_gemm_mode(mode)
            ms = timeit(lambda: ops.gemm(dy, x, a_mn=True, b_mn=True))
            print(f"{name:8s} [{m} x {h} x K {T}] {label}: {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s", flush=True)
    lib().lynx_op_gemm_mode(-1)


if __name__ == "__main__":
    main()
