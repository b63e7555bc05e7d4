LYNX_LN_PARTS=8 timeout 300 python -m pytest tests/test_ops_gpu.py -x -q -k "layernorm or ln" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_ops_gpu.py -x -q -k "layernorm or ln" 2>&1 | tail -1
for w in 2 4 8; do LYNX_LN_PARTS=$w timeout 120 python tools/bench_elem.py 2>&1 | grep ln_fwd; done
