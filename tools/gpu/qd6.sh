timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "speculative or cfg0 or cfg3_small or appendix or cfg1" > gpurun_out/t21.log 2>&1; tail -12 gpurun_out/t21.log
bash tools/gpu/qd5.sh
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
