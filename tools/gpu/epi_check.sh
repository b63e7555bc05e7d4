timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -k "gemm" 2>&1 | tail -3
timeout 600 python tools/step_ops.py --steps 5 --out gpurun_out/step_ops2.json 2>&1 | head -24
