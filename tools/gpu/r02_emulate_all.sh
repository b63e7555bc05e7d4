# Round-2 stage emulations (one TP rank per stage alone on one B200; all-reduces and pipeline stalls as
# stand-ins), HEU vs the elided floor vs Megatron full / selective, for every BASELINE multi-GPU config.
set -u
E="python tools/emulate_stage.py"
V="heu,elided,full_recompute,selective"
timeout 1200 $E --model 7b --stages 0,1,2,3 --variants $V --out gpurun_out/r02_emulate_7b_tp2pp4_168gb.json > gpurun_out/r02_e7.log 2>&1; echo e7=$?
timeout 1200 $E --model 1.3b --stages 0,1,2,3 --budget-gb 24 --variants $V --out gpurun_out/r02_emulate_1.3b_tp2pp4_24gb.json > gpurun_out/r02_e13.log 2>&1; echo e1.3=$?
timeout 1200 $E --model 13b --stages 0,1 --budget-gb 40 --variants $V --out gpurun_out/r02_emulate_13b_tp4pp2_40gb.json > gpurun_out/r02_e13b.log 2>&1; echo e13=$?
timeout 1200 $E --model 20b --tp 8 --pp 1 --stages 0 --budget-gb 80 --variants $V --out gpurun_out/r02_emulate_20b_tp8pp1_80gb.json > gpurun_out/r02_e20a.log 2>&1; echo e20a=$?
timeout 1200 $E --model 20b --tp 4 --pp 2 --stages 0,1 --budget-gb 80 --variants $V --out gpurun_out/r02_emulate_20b_tp4pp2_80gb.json > gpurun_out/r02_e20b.log 2>&1; echo e20b=$?
timeout 1500 $E --model 7b --stages 0,1,2,3 --budget-gb 80 --variants heu,elided,full_recompute --out gpurun_out/r02_emulate_7b_tp2pp4_80gb.json > gpurun_out/r02_e780.log 2>&1; echo e7_80=$?
