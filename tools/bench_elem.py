"""HBM-bound operators of the GPT block at the GPT-7B bench shape (T=65536 tokens, h=4096).

    python tools/bench_elem.py [T h]
Prints ms and achieved GB/s (algorithmic bytes: every tensor read or written once)
against the measured copy bandwidth in MEASURED_PEAKS.json.
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402


def timeit(fn, iters=5):
    for _ in range(2):
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
    T, h = (int(x) for x in sys.argv[1:3]) if len(sys.argv) > 2 else (65536, 4096)
    peak = None
    p = os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p)).get("hbm_gbs")
    dev, bf = "cuda", torch.bfloat16
    x = torch.randn(T, h, device=dev).to(bf)
    y = torch.randn(T, h, device=dev).to(bf)
    g = torch.ones(h, device=dev, dtype=bf)
    b = torch.zeros(h, device=dev, dtype=bf)
    f = torch.randn(T, 4 * h, device=dev).to(bf)
    y2, mean, rstd = ops.layernorm_fwd(x, g, b)
    dg, db, acc = (torch.zeros(h, device=dev), torch.zeros(h, device=dev), torch.zeros(4 * h, device=dev))
    e = 2 * T * h  # bytes of one [T, h] bf16 tensor
    cases = [
        ("ln_fwd", lambda: ops.layernorm_fwd(x, g, b), 2 * e),
        ("ln_bwd(+dres)", lambda: ops.layernorm_bwd(y, x, g, mean, rstd, dg, db, dres=y2), 4 * e),
        ("bias_dropout_residual", lambda: ops.bias_dropout_residual(y, g, x, 0.1, 1, 2), 3 * e),
        ("dropout_bwd", lambda: ops.dropout_bwd(y, 0.1, 1, 2), 2 * e),
        ("gelu_fwd [T,4h]", lambda: ops.gelu_fwd(f), 8 * e),
        ("gelu_bwd [T,4h]", lambda: ops.gelu_bwd(f, f), 12 * e),
        ("column_sum [T,4h]", lambda: ops.column_sum_acc(f, acc), 4 * e),
        ("column_sum [T,h]", lambda: ops.column_sum_acc(y, dg), e),
        ("dropout_bwd_colsum", lambda: ops.dropout_bwd_colsum(y, dg, 0.1, 1, 2), 2 * e),
    ]
    for name, fn, nbytes in cases:
        t = timeit(fn)
        gbs = nbytes / t / 1e6
        frac = f" {gbs / peak:5.2f} of {peak:.0f}" if peak else ""
        print(f"{name:24s} {t:7.3f} ms {gbs:8.1f} GB/s{frac}", flush=True)


if __name__ == "__main__":
    main()
