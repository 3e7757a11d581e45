set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gpu_tests7.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/gpu_tests7.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench7.log 2>&1; echo "bench rc $?"; tail -c 600 gpurun_out/bench7.log
timeout 600 python tools/bench_proj_sweep.py --ranks 16,19,20,21,24,32,64,128 > gpurun_out/proj_sweep7.json 2> gpurun_out/proj_sweep7.err; echo "sweep rc $?"
TTG_DEBUG=1 timeout 300 python tools/profile_window.py --skip 18 --steps 2 > gpurun_out/pw_debug7.log 2>&1; grep "eig_top" gpurun_out/pw_debug7.log | tail -8
timeout 900 python tools/bench_configs.py --cfg 1,2 --increments 50 > gpurun_out/cfg12_7.json 2> gpurun_out/cfg12_7.err; echo "cfg rc $?"
