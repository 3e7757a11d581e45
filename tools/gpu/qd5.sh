for v in "" "TTG_NO_SPEC=1" "TTG_NO_TAIL=1" "TTG_NO_DECIDE=1"; do
  env $v python tools/bench_configs.py --cfg 1 > gpurun_out/c1.json 2> gpurun_out/c1.err
  python -c "
import json; d=json.load(open('gpurun_out/c1.json'))
for r in d['rows']: print('$v', r['algo'], round(r['ms_per_update'],3), round(r['GBs_ingested'],1), [(k['name'],k['launches'],round(k['ms'],1)) for k in r['top_kernels'][:4]])"
done
