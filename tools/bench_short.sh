# quick bench: value, ms/step, per-step device ms, top kernels (used during tuning)
python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --kernels-out gpurun_out/kk.json > gpurun_out/bb.log 2>&1
tail -1 gpurun_out/bb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],2), [s['device_ms'] for s in d['steps_detail']])"
python -c "
import json; k=json.load(open('gpurun_out/kk.json'))
for x in k[:${TOPK:-8}]: print(round(x['ms'],3), x['launches'], x['name'])
"
