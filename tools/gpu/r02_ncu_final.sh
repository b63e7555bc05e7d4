#!/bin/bash
# Round-2 final ncu evidence: launch list of one bench step (plan replayed from the final bench line's op
# times) and --set full captures of the three attention kernels at the GPT-7B layer shape.
set -u
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-crosscheck --no-stage-emulation --op-times profiles/r02_bench_n1_final.json"
timeout 900 $CMD > gpurun_out/r02f_plain.json 2> gpurun_out/r02f_plain.err; echo plain_rc=$?
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_final.csv $CMD > gpurun_out/r02f_launches.log 2>&1; echo launches_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:attn_fwd2_tc_kernel" -s 2 -c 1 -o gpurun_out/r02_attn128_fwd2_final -f python tools/bench_attn.py 16 2048 32 128 > gpurun_out/r02f_ncu_fwd.log 2>&1; echo ncu_fwd_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:attn_(dkdv|dq)_tc_kernel" -s 2 -c 2 -o gpurun_out/r02_attn128_bwd_final -f python tools/bench_attn.py 16 2048 32 128 > gpurun_out/r02f_ncu_bwd.log 2>&1; echo ncu_bwd_rc=$?
python tools/ncu_summary.py gpurun_out/r02_attn128_fwd2_final.ncu-rep > gpurun_out/r02_attn128_final_summary.txt
python tools/ncu_summary.py gpurun_out/r02_attn128_bwd_final.ncu-rep >> gpurun_out/r02_attn128_final_summary.txt
cat gpurun_out/r02_attn128_final_summary.txt
