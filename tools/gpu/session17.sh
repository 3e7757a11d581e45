set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t17.log 2>&1; tail -3 gpurun_out/t17.log
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
