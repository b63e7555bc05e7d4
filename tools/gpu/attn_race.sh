timeout 300 python tools/attn_race.py 1000 1 1024 1 64
timeout 300 python tools/attn_race.py 300 1 256 4 64
timeout 300 python tools/attn_race.py 300 2 640 2 128
for i in 1 2 3 4 5 6; do timeout 120 python -m pytest tests/test_ops_gpu.py -x -q -k "test_attention" 2>&1 | tail -1; done
timeout 120 python tools/bench_attn.py 2>&1 | tail -3
