set -x
N_INC=5 timeout 900 python tools/gpu/debug_cfg2.py > gpurun_out/dbg_cfg2.log 2>&1; echo rc $?
TTG_NO_TALL=1 N_INC=5 timeout 900 python tools/gpu/debug_cfg2.py > gpurun_out/dbg_cfg2_notall.log 2>&1; echo rc $?
