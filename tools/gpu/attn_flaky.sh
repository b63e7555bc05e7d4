for i in $(seq 1 12); do timeout 120 python -m pytest tests/test_ops_gpu.py -x -q -k "test_attention" 2>&1 | grep -E "^FAILED|^E  .*assert|passed|failed" | head -3; done
