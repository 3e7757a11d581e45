set -x
N_INC=5 timeout 900 python tools/gpu/debug_cfg2.py > gpurun_out/dbg_cfg2.log 2>&1; echo rc $?; tail -4 gpurun_out/dbg_cfg2.log
timeout 1200 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 800 > gpurun_out/fs6.log 2>&1; echo "fullsize rc $?"; tail -4 gpurun_out/fs6.log
timeout 900 python tools/bench_configs.py --cfg 2 --increments 50 > gpurun_out/cfg2_6.json 2> gpurun_out/cfg2_6.err; echo "cfg2 rc $?"; tail -c 1200 gpurun_out/cfg2_6.json
