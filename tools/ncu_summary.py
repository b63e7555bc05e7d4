"""Key metrics per kernel from an ncu report: python tools/ncu_summary.py report.ncu-rep [name-regex]

Tensor / shared / XU pipe activity, issue activity, DRAM bytes, duration, registers and the top
warp-stall reasons (ratio per issued instruction)."""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts (tc) %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__registers_per_thread", "registers"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        if pat and not pat.search(name):
            continue
        print(f"== {name[:90]}")
        for k, label in KEYS:
            if k in col:
                print(f"   {label:24s} {r[col[k]]} {units[col[k]]}")
        stalls = [(float(r[i] or 0), h) for h, i in col.items()
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        top = sorted(stalls, reverse=True)[:5]
        print("   stalls/issue           " + ", ".join(
            f"{h.split('stalled_')[1].split('_per_issue')[0]} {v:.2f}" for v, h in top))


if __name__ == "__main__":
    main()
