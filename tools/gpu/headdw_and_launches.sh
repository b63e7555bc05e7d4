for m in -1 1; do LYNX_GEMM_MODE=$m timeout 60 python tools/gemm_sustained.py 65536 headdw; LYNX_GEMM_MODE=$m timeout 60 python tools/gemm_sustained.py 65536 headfwd; done
timeout 60 python tools/gemm_sustained.py 65536 headdw cublas
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-crosscheck > gpurun_out/b112.json 2> gpurun_out/b112.err; echo bench_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b_r4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-crosscheck > gpurun_out/ncu112.log 2>&1; echo ncu_rc=$?
