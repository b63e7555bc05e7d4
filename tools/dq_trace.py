"""Item transitions of the persistent dQ (KERNEL=dq, default) or dK/dV (KERNEL=dkdv) kernel (CTA 0): LYNX_BUILD_TRACE=1 build, then
python tools/dq_trace.py [B S H D]. Tags per item k: 8 rows start the item, 7 rows handed the last
dS, 9 rows saw fin, 11 rows wrote dQ, 10 MMA saw the item's Q / dO staged, 12 MMA committed fin,
13 rows got the item's first S."""
import os
import re
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, ".")
    from paper_2406_08756_b200 import ops
    B, S, H, D = (int(x) for x in sys.argv[2:6])
    qkv = (torch.randn(B * S, 3 * H * D, device="cuda") * 0.5).bfloat16()
    dout = torch.randn(B * S, H * D, device="cuda").bfloat16()
    out, lse = ops.attention_fwd(qkv, B, S, H, D)
    torch.cuda.synchronize()
    print("=== BWD", flush=True)
    ops.attention_bwd(qkv, out, dout, lse, B, S, H, D)
    torch.cuda.synchronize()
    sys.exit(0)
args = sys.argv[1:5] if len(sys.argv) > 4 else ["16", "2048", "32", "128"]
txt = subprocess.run([sys.executable, __file__, "--child", *args], capture_output=True, text=True).stdout
lines = re.findall(r"^T (\d+) (\d+) (\d+)$", txt.split("=== BWD", 1)[1], re.M)
which = os.environ.get("KERNEL", "dq")
lines = lines[len(lines) // 2:] if which == "dq" else lines[:len(lines) // 2]  # dK/dV dumps first, then dQ
ev = {}
for t, j, c in lines:
    ev.setdefault(int(t), {})[int(j)] = int(c)
t0 = ev[8][0]
print(" k     start last_arr fin_seen   staged   synced epi_done    mma_q  first_S  mma_fin")
for k in range(60):
    if k not in ev[13] or ev[13][k] == 0 or (k > 0 and ev[13][k] <= ev[13][k - 1]):
        break
    g = lambda t: ev[t][k] - t0
    print(f"{k:2d} {g(8):8d} {g(7):8d} {g(9):8d} {g(15):8d} {g(5):8d} {g(11):8d} {g(10):8d} {g(13):8d} {g(12):8d}")
