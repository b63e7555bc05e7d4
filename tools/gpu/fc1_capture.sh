timeout 900 python -m pytest tests/test_ops_gpu.py -x -q -k "gemm" 2>&1 | tail -1
timeout 120 python tools/gemm_one.py > gpurun_out/g2.log 2>&1; echo gemm_one_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 1 -c 1 -o gpurun_out/ncu_fc1_r5 -f python tools/gemm_one.py > gpurun_out/ncu_fc1.log 2>&1; echo ncu_rc=$?
