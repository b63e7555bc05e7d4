timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t148.log 2>&1; tail -1 gpurun_out/t148.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench148.json 2>gpurun_out/bench148.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench148.json').read().strip().splitlines()[-1]); print(d['value'], d['step_ms_each'], d['exposed_recompute_ms_per_iter'], d['clocks']['sm_mhz'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['recompute']['baselines']['elided']['iteration_ms'])"
timeout 600 python bench.py --impl reference > gpurun_out/ref148.json 2>/dev/null; tail -c 200 gpurun_out/ref148.json
