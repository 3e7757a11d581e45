set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/gpu_tests8.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/gpu_tests8.log
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench8.log 2>&1; echo "bench rc $?"; tail -c 300 gpurun_out/bench8.log
TTG_DEBUG=1 timeout 300 python tools/profile_window.py --skip 18 --steps 2 > gpurun_out/pw_debug8.log 2>&1; grep "eig_top" gpurun_out/pw_debug8.log | tail -8
timeout 600 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pw_launches8.csv python tools/profile_window.py --skip 18 --steps 2 > gpurun_out/pw_ncu8.log 2>&1; echo "ncu rc $?"
TTG_PWS_LOW=1 timeout 600 python tools/bench_proj_sweep.py --ranks 16,19,20,21,24,32 > gpurun_out/proj_sweep8_pws.json 2> gpurun_out/proj_sweep8_pws.err; echo "sweep rc $?"
