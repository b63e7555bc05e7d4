# Round-2 ncu evidence (one gpurun call): launch list of one bench step (plan replayed from the measured
# run's op times, profiles/r02_bench_n1.json) and --set full captures of the FC1 forward GEMM and the
# head_dim-112 attention backward kernels.
set -u
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-crosscheck --no-stage-emulation --op-times profiles/r02_bench_n1.json"
timeout 900 $CMD > gpurun_out/r02_ncu_plain.json 2> gpurun_out/r02_ncu_plain.err; echo plain_rc=$?
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_ncu_launches.log 2>&1; echo launches_rc=$?
timeout 300 python tools/bench_attn.py 8 2048 8 112 > gpurun_out/r02_attn112.log 2>&1; echo attn_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:attn_(dkdv|dq)_tc_kernel" -s 2 -c 2 -o gpurun_out/r02_attn112_bwd -f python tools/bench_attn.py 8 2048 8 112 > gpurun_out/r02_ncu_attn.log 2>&1; echo ncu_attn_rc=$?
