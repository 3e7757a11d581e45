timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tail_shapes or speculative" > gpurun_out/t22.log 2>&1; tail -15 gpurun_out/t22.log
