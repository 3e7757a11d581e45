# ncu launch list of one skip + one update step at the ranks the bench reaches (NVTX window)
set -x
python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/r02_window.log 2>&1 && \
ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_window_r21_launches.csv python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/r02_window_ncu.log 2>&1; echo "rc $?"; tail -2 gpurun_out/r02_window.log
