timeout 600 python -m pytest tests/test_gpu_io_metrics.py -x -q 2>&1 | tail -2
for v in "TTG_RRE_DFMA=1" ""; do
env $v python tools/bench_io.py > gpurun_out/r02_io_bench.json 2> gpurun_out/r02_io.err; python -c "
import json; d=json.load(open('gpurun_out/r02_io_bench.json')); print('$v', round(d['rre']['value'],1), d['rre']['rre'], d['rre']['kernel']['ms_per_launch'], round(d['rre']['kernel']['roofline']['frac'],3))"
done
