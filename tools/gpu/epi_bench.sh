timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -k "gelu or gemm or resid" 2>&1 | tail -2
for sh in dgelu_plain dgelu fc2_plain fc2res; do timeout 60 python tools/gemm_sustained.py 65536 $sh; done
for sh in dgelu fc2res; do LYNX_GEMM_AUX_TMA=0 timeout 60 python tools/gemm_sustained.py 65536 $sh; done
timeout 600 python tools/step_ops.py --steps 4 --out gpurun_out/step_ops3.json 2>&1 | head -20
