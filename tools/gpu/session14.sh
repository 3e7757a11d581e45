set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t14.log 2>&1; tail -5 gpurun_out/t14.log
