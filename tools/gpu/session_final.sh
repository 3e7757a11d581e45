# Round-end measurement set (one call): bench line, reference arm, per-kernel table,
# ncu launch list of the same bench command, other configs, companion sweep, io bench.
set -x
python bench.py --steps 20 --warmup 5 --kernels-out gpurun_out/r02_kernels.json > gpurun_out/r02_bench.log 2>&1; echo "bench rc $?"
tail -1 gpurun_out/r02_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['roofline']['step_roofline_frac'],3), d['e2e']['value'] if d['e2e'] else None, d['gpu_launches'])"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref.log 2>&1; tail -1 gpurun_out/r02_ref.log | cut -c1-300
python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02_ncu.log 2>&1; echo "ncu rc $?"
timeout 900 python tools/bench_configs.py > gpurun_out/r02_configs.json 2> gpurun_out/r02_configs.err; echo "configs rc $?"
timeout 600 python tools/bench_proj_sweep.py > gpurun_out/r02_proj_sweep.json 2> gpurun_out/r02_proj_sweep.err; echo "sweep rc $?"
timeout 600 python tools/bench_io.py > gpurun_out/r02_io_bench.json 2> gpurun_out/r02_io.err; echo "io rc $?"
torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu --no-e2e --force-dist > gpurun_out/r02_bench_nccl1.log 2>&1; tail -1 gpurun_out/r02_bench_nccl1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nccl world 1:', round(d['value'],1))"
