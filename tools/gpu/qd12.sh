for v in "" "TTG_NO_SPEC=1"; do
  env $v python tools/bench_configs.py --cfg 1,2 > gpurun_out/c1.json 2> gpurun_out/c1.err
  python -c "
import json; d=json.load(open('gpurun_out/c1.json'))
for r in d['rows']: print('$v', r['cfg'], r['algo'], round(r['ms_per_update'],3), round(r['GBs_ingested'],1))"
done
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
