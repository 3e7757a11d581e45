set -x
python tools/make_fullsize_fixtures.py cfg1 --out tests/golden > gpurun_out/fx1.log 2>&1; echo "fx1 rc $?"
python tools/make_fullsize_fixtures.py cfg2 --out tests/golden > gpurun_out/fx2.log 2>&1; echo "fx2 rc $?"
mkdir -p gpurun_out/golden && cp tests/golden/cfg1_full_*.npz tests/golden/cfg2_full_*.npz gpurun_out/golden/
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 800 > gpurun_out/fs4.log 2>&1; echo "fullsize rc $?"; tail -4 gpurun_out/fs4.log
timeout 300 python tools/profile_window.py --skip 18 --steps 2 > gpurun_out/pw_plain.log 2>&1; cat gpurun_out/pw_plain.log
TTG_DEBUG=1 timeout 300 python tools/profile_window.py --skip 18 --steps 2 > gpurun_out/pw_debug.log 2>&1; grep -c eig gpurun_out/pw_debug.log
timeout 600 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pw_launches.csv python tools/profile_window.py --skip 18 --steps 2 > gpurun_out/pw_ncu.log 2>&1; echo "ncu rc $?"
timeout 600 python tools/bench_proj_sweep.py --ranks 16,17,18,19,20,21,22,23,24,32,64,128 > gpurun_out/proj_sweep4.json 2> gpurun_out/proj_sweep4.err; echo "sweep rc $?"
timeout 900 python tools/bench_configs.py --cfg 2 --increments 50 > gpurun_out/cfg2_4.json 2> gpurun_out/cfg2_4.err; echo "cfg2 rc $?"; tail -c 600 gpurun_out/cfg2_4.json
