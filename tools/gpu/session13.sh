set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t13.log 2>&1; tail -5 gpurun_out/t13.log
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
timeout 900 python tools/bench_configs.py --cfg 1 > gpurun_out/r02_configs_b.json 2> gpurun_out/r02_configs_b.err; python -c "
import json; d=json.load(open('gpurun_out/r02_configs_b.json'))
for r in d['rows']: print(r['cfg'],r['algo'],round(r['ms_per_update'],3),round(r['GBs_ingested'],1),r['final_ranks'])"
