timeout 900 python tools/emulate_stage.py --model 7b --stages 0,1,2,3 --out gpurun_out/emulate_7b.json 2>&1 | tail -4
timeout 900 python tools/emulate_stage.py --model 7b --budget-gb 80 --stages 0,3 --out gpurun_out/emulate_7b_80gb.json 2>&1 | tail -2
timeout 900 python tools/emulate_stage.py --model 13b --budget-gb 40 --stages 0,1 --out gpurun_out/emulate_13b_40gb.json 2>&1 | tail -2
