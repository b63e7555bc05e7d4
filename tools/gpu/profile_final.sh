timeout 120 python tools/gemm_one.py > gpurun_out/g1.log 2>&1; echo gemm_one_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 8 -c 1 -o gpurun_out/ncu_dgelu -f python tools/gemm_one.py > gpurun_out/ncu_dgelu.log 2>&1; echo ncu_full_rc=$?
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-crosscheck > gpurun_out/b121.json 2> gpurun_out/b121.err; echo bench_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b_r5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-crosscheck > gpurun_out/ncu121.log 2>&1; echo ncu_rc=$?
