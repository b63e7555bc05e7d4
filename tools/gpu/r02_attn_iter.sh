#!/bin/bash
# attention iteration: parity tests, timings at the 7B and 1.3B shapes, then a dK/dV clock64 trace
set -x
python -m pytest tests/test_ops_gpu.py -q -x -k "attention" 2>&1 | tail -3
python tools/bench_attn.py 16 2048 32 128
python tools/bench_attn.py 8 2048 8 112
touch paper_2406_08756_b200/csrc/ops_attention_tc.cu; LYNX_BUILD_TRACE=1 python -m paper_2406_08756_b200.build > /dev/null 2>&1
LYNX_ATTN_FWD_TILES=3 python tools/attn_trace.py 16 2048 32 128 > gpurun_out/attn_trace_fwd3.txt 2>&1; python tools/attn_trace.py 16 2048 32 128 > gpurun_out/attn_trace_dkdv.txt 2>&1
grep -A17 "== fwd2" gpurun_out/attn_trace_dkdv.txt; grep -A12 "== dK" gpurun_out/attn_trace_dkdv.txt; grep -A12 "== dQ" gpurun_out/attn_trace_dkdv.txt
grep -A40 "== fwd2" gpurun_out/attn_trace_fwd3.txt | head -42
