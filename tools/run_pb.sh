python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -q -m gpu -x > gpurun_out/parity.log 2>&1; tail -2 gpurun_out/parity.log
for o in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --kernels-out gpurun_out/kk.json > gpurun_out/bb.log 2>&1; tail -1 gpurun_out/bb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],2), [s['device_ms'] for s in d['steps_detail']])"; done
python -c "
import json; k=json.load(open('gpurun_out/kk.json'))
for x in k[:14]: print(round(x['ms'],3), x['launches'], round(x['bytes']/x['ms']/1e9/x['launches']*x['launches'],1) if x['ms'] else 0, x['name'])
"
