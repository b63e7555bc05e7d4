timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_executor_gpu.py -x -q 2>&1 | tail -2
timeout 600 python tools/step_ops.py --steps 4 --out gpurun_out/step_ops4.json 2>&1 | head -24
