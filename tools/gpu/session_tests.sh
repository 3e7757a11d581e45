set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t17.log 2>&1; tail -3 gpurun_out/t17.log
