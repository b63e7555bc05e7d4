#!/bin/bash
# Stage emulations with stand-in all-reduces that sleep (passes 0) vs stream their buffer through HBM
# (passes 1 at TP2, 2 at TP4: a ring all-reduce's local traffic and SM occupancy), same box back to back
set -u
E="python tools/emulate_stage.py"
V="heu,elided"
for p in 0 1; do
  timeout 1500 $E --model 7b --stages 0 --budget-gb 80 --variants $V --standin-passes $p --out gpurun_out/r02_emulate_7b_80gb_p$p.json > gpurun_out/r02_et7_$p.log 2>&1; echo 7b_p$p=$?
done
for p in 0 2; do
  timeout 1500 $E --model 13b --stages 0 --budget-gb 40 --variants $V --standin-passes $p --out gpurun_out/r02_emulate_13b_40gb_p$p.json > gpurun_out/r02_et13_$p.log 2>&1; echo 13b_p$p=$?
done
python - <<'PY'
import json
for f in ("r02_emulate_7b_80gb_p0", "r02_emulate_7b_80gb_p1", "r02_emulate_13b_40gb_p0", "r02_emulate_13b_40gb_p2"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e:
        print(f, "missing", e); continue
    for s, row in d["stages"].items():
        h = row.get("heu", {}); el = row.get("elided", {})
        print(f, s, {k: round(h.get(k), 1) for k in ("iteration_ms", "comm_ms", "exposed_recompute_ms",
                                                     "recompute_overlapped_ms", "sm_mhz_median")},
              "elided", round(el.get("iteration_ms"), 1), "crosscheck", round(h["iteration_ms"] - el["iteration_ms"], 1))
PY
