"""Per-tile clock64 timeline of the attention backward dK/dV kernel (CTA 0, the longest key tile).

    LYNX_BUILD_TRACE=1 python -m paper_2406_08756_b200.build && python tools/attn_trace.py [B S H D] > trace.txt
Then the dQ kernel's, same tags. Tags (ops_attention_tc.cu ATRACE): 0 producer issues Q/dO(i), 1 MMA issues S^T/dP^T(i), 2 MMA got
P^T/dS^T(i) and issues dV/dK(i), 3 rows got S^T/dP^T(i), 4 rows computed(i), 6 rows handed P^T/dS^T(i).
"""
import re
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, ".")
    from paper_2406_08756_b200 import ops
    from paper_2406_08756_b200._native import lib
    B, S, H, D = (int(x) for x in sys.argv[2:6])
    lib().lynx_op_attention_mode(-1)
    qkv = (torch.randn(B * S, 3 * H * D, device="cuda") * 0.5).bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    print("=== FWD", flush=True)
    out, lse = ops.attention_fwd(qkv, B, S, H, D)
    torch.cuda.synchronize()
    print("=== BWD", flush=True)
    ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
    torch.cuda.synchronize()
    sys.exit(0)

args = sys.argv[1:5] if len(sys.argv) > 4 else ["16", "2048", "32", "128"]
txt = subprocess.run([sys.executable, __file__, "--child", *args], capture_output=True, text=True).stdout
fwd_part, part = txt.split("=== FWD", 1)[1].split("=== BWD", 1)
fl = re.findall(r"^T (\d+) (\d+) (\d+)$", fwd_part, re.M)
if fl:  # two-tile forward: 0 S0 issue, 1 PV0 issue, 2/3 softmax0 start/arrive, 4/5 softmax1, 6 PV1, 7 S1
    ev = {}
    for t, j, c in fl:
        ev.setdefault(int(t), {})[int(j)] = int(c)
    n = max(ev[2]) + 1
    t0 = min(v for t in ev for v in ev[t].values() if v)
    print("== fwd2: j   S0   PV0  sm0s  sm0a  sm1s  sm1a   PV1    S1 | sm0_dur sm1_dur PV0_gap | sm0: ld max exp pack st")
    for i in range(n):
        g = lambda t: ev.get(t, {}).get(i, t0) - t0
        print(f"{i:4d} " + " ".join(f"{g(t):6d}" for t in (0, 1, 2, 3, 4, 5, 6, 7)) +
              f" | {g(3) - g(2):6d} {g(5) - g(4):6d} {(ev[1][i] - ev[1][i - 1]) if i else 0:6d} | "
              f"{g(8) - g(2):5d} {g(9) - g(8):5d} {g(10) - g(9):5d} {g(11) - g(10):5d} {g(12) - g(11):5d}")
lines = re.findall(r"^T (\d+) (\d+) (\d+)$", part, re.M)
if not lines:
    print(txt[-2000:])
    sys.exit(1)
half = len(lines) // 2  # 16 tags each  # the dK/dV kernel's dump, then the dQ kernel's (same CTA shape: n tiles each)
for name, chunk in (("dK/dV", lines[:half]), ("dQ", lines[half:])):
    ev = {}
    for t, j, c in chunk:
        ev.setdefault(int(t), {})[int(j)] = int(c)
    n = max(ev[3]) + 1
    t0 = min(v for t in (0, 1, 2, 3, 4, 6) for v in ev[t].values())
    print(f"== {name}: tile  prod  mmaS  mmaG  rows0 rowsC rowsA | rows_dur wait_for_S  mmaG_gap")
    for i in range(n):
        g = lambda t: ev.get(t, {}).get(i, t0) - t0
        print(f"{i:4d} {g(0):6d} {g(1):6d} {g(2):6d} {g(3):6d} {g(4):6d} {g(6):6d} | {g(6) - g(3):7d} "
              f"{(ev[3][i] - ev[6][i - 1]) if i else 0:9d} {(ev[2][i] - ev[2][i - 1]) if i else 0:9d}")
