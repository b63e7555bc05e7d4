"""Back-to-back GEMM for ~2 s (power-capped steady state): TFLOP/s and median SM clock.

    LYNX_GEMM_GROUP=G python tools/gemm_sustained.py [T] [shape]   shape: fc1 | fc2 | dx | dw
"""
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2406_08756_b200 import ops  # noqa: E402


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    shape = sys.argv[2] if len(sys.argv) > 2 else "fc1"
    h = 4096
    if shape == "fc1":
        a, b, kw, fl = torch.randn(T, h), torch.randn(4 * h, h), {}, 2.0 * T * 4 * h * h
    elif shape == "fc2":
        a, b, kw, fl = torch.randn(T, 4 * h), torch.randn(h, 4 * h), {}, 2.0 * T * 4 * h * h
    elif shape == "dx":
        a, b, kw, fl = torch.randn(T, 4 * h), torch.randn(4 * h, h), {"b_mn": True}, 2.0 * T * 4 * h * h
    elif shape in ("dgelu", "dgelu_plain"):  # FC2 dX with (or without) the fused GeLU backward
        a, b, kw, fl = torch.randn(T, h), torch.randn(h, 4 * h), {"b_mn": True}, 2.0 * T * 4 * h * h
    elif shape in ("fc2res", "fc2_plain"):  # FC2 forward with (or without) the fused bias-dropout-residual
        a, b, kw, fl = torch.randn(T, 4 * h), torch.randn(h, 4 * h), {}, 2.0 * T * 4 * h * h
    elif shape == "headdw":  # LM-head weight gradient per 4096-token chunk: [V, h] += logits^T X
        V, C = 50304, 4096
        a, b, kw, fl = torch.randn(C, V), torch.randn(C, h), {"a_mn": True, "b_mn": True}, 2.0 * V * h * C
    elif shape == "headfwd":  # LM-head logits per chunk: [C, V] = X W^T
        V, C = 50304, 4096
        a, b, kw, fl = torch.randn(C, h), torch.randn(V, h), {}, 2.0 * V * h * C
    else:
        a, b, kw, fl = torch.randn(T, 4 * h), torch.randn(T, h), {"a_mn": True, "b_mn": True}, 2.0 * T * 4 * h * h
    a, b = a.cuda().bfloat16(), b.cuda().bfloat16()
    if shape == "dw":
        out = torch.zeros(4 * h, h, device="cuda")
        kw["epi"] = ops.EPI_F32
    elif shape == "headdw":
        out = torch.zeros(50304, h, device="cuda")
        kw["epi"] = ops.EPI_F32
    else:
        out = None
    use_cublas = len(sys.argv) > 3 and sys.argv[3] == "cublas"
    if use_cublas:  # yardstick: torch.matmul with the same operand layouts
        A = a.t() if kw.get("a_mn") else a
        B = b if kw.get("b_mn") else b.t()
        kw = {}

        def run():
            torch.matmul(A, B)
    elif shape == "dgelu":
        x = torch.randn(T, 4 * h, device="cuda").bfloat16()

        def run():
            ops.gemm_gelu_bwd(a, b, x, b_mn=True)
    elif shape == "fc2res":
        res = torch.randn(T, h, device="cuda").bfloat16()

        def run():
            ops.gemm_residual(a, b, res, p=0.1, seed=1, stream_id=2)
    else:
        def run():
            ops.gemm(a, b, out=out, **kw)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    clocks = []
    stop = threading.Event()

    def sample():
        try:
            import pynvml
            pynvml.nvmlInit()
            hd = pynvml.nvmlDeviceGetHandleByIndex(0)
            while not stop.is_set():
                clocks.append(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM))
                time.sleep(0.02)
        except Exception:
            pass

    th = threading.Thread(target=sample, daemon=True)
    th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    s.record()
    t0 = time.time()
    while time.time() - t0 < 2.0:
        for _ in range(5):
            run()
        n += 5
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    ms = s.elapsed_time(e) / n
    clocks.sort()
    med = clocks[len(clocks) // 2] if clocks else None
    print(f"{'cublas' if use_cublas else 'lynx'} {shape} T={T} ms={ms:.3f} TFLOP/s={fl / ms / 1e9:.1f} sm_mhz_median={med}", flush=True)


if __name__ == "__main__":
    main()
