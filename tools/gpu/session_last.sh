set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t_last.log 2>&1; tail -3 gpurun_out/t_last.log
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default bench', d['steps'], d['warmup'], round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['step_roofline_frac'],3), d['e2e']['value'], d['gpu_launches'], d['clocks'])"
