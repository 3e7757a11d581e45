set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or cfg0 or speculative or ranks_17 or heuristic or project or determinism" > gpurun_out/t18.log 2>&1; tail -3 gpurun_out/t18.log
for v in 1 0; do
  if [ $v = 1 ]; then export TTG_NO_TAIL=1; else unset TTG_NO_TAIL; fi
  python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_TAIL=$v', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
done
