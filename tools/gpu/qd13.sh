python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_io_metrics.py -x -q 2>&1 | tail -2
python tools/bench_io.py > gpurun_out/r02_io_bench.json 2> gpurun_out/r02_io.err; python -c "
import json; d=json.load(open('gpurun_out/r02_io_bench.json')); print(d['rre']['value'], d['rre']['kernel'])"
