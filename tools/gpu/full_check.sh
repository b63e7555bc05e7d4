timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t120.log 2>&1; tail -2 gpurun_out/t120.log
timeout 900 python bench.py > gpurun_out/bench120.json 2>gpurun_out/bench120.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench120.json').read().strip().splitlines()[-1]); print(d['value'], d['step_ms_each'], d['exposed_recompute_ms_per_iter'], d['clocks'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['recompute']['baselines']['elided']['iteration_ms'], d['memory']['oom_retries'])"
