timeout 600 python tools/emulate_stage.py --model 7b --tp 2 --pp 1 --microbatches 2 --stages 0 --out gpurun_out/emulate_7b_tp2pp1.json 2>&1 | tail -1
timeout 900 python tools/emulate_stage.py --model 7b --tp 2 --pp 2 --microbatches 4 --stages 0,1 --out gpurun_out/emulate_7b_tp2pp2.json 2>&1 | tail -2
