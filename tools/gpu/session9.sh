set -x
timeout 900 python tools/bench_configs.py > gpurun_out/r02_configs.json 2> gpurun_out/r02_configs.err; echo "configs rc $?"; tail -c 1500 gpurun_out/r02_configs.json
timeout 600 python tools/bench_proj_sweep.py > gpurun_out/r02_proj_sweep.json 2> gpurun_out/r02_proj_sweep.err; echo "sweep rc $?"; tail -c 1200 gpurun_out/r02_proj_sweep.json
timeout 600 python tools/bench_io.py > gpurun_out/r02_io_bench.json 2> gpurun_out/r02_io.err; echo "io rc $?"; tail -c 600 gpurun_out/r02_io_bench.json
timeout 300 python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/r02_pw.log 2>&1; tail -3 gpurun_out/r02_pw.log
timeout 600 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_pw_launches.csv python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/r02_pw_ncu.log 2>&1; echo "ncu rc $?"
