#!/bin/bash
# Round-2 end-of-session check: full GPU suite, smoke, default bench line (N = 1)
set -u
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_final.log 2>&1; tail -2 gpurun_out/r02_gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke_final.log 2>&1; tail -1 gpurun_out/r02_smoke_final.log
timeout 1500 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench_final.err; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02_bench_final.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "ms_per_step", "exposed_recompute_ms_per_iter", "exposed_recompute_crosscheck_ms")})
print("clocks", d["clocks"], "roofline", d["roofline"], "e2e", d["e2e"]["value"])
PY
