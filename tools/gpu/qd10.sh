timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py -x -q -k "cfg1 or speculative or cfg0 or wide or ranks_17 or high_ranks" > gpurun_out/t23.log 2>&1; tail -5 gpurun_out/t23.log
python tools/bench_configs.py --cfg 1 > gpurun_out/c1.json 2> gpurun_out/c1.err
python -c "
import json; d=json.load(open('gpurun_out/c1.json'))
for r in d['rows']: print(r['algo'], round(r['ms_per_update'],3), round(r['GBs_ingested'],1), [(k['name'],k['launches'],round(k['ms'],1)) for k in r['top_kernels'][:5]])"
