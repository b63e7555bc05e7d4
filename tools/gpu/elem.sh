timeout 300 python -m pytest tests/test_ops_gpu.py -x -q -k "column or dropout" 2>&1 | tail -1
timeout 120 python tools/bench_elem.py 2>&1
