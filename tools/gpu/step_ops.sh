timeout 600 python tools/step_ops.py --steps 6 --out gpurun_out/step_ops.json
