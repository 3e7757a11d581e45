TTG_DECIDE_TWICE=1 TTG_NO_SPEC=1 TTG_DEBUG=1 timeout 300 python tools/profile_window.py --skip 17 --steps 1 > gpurun_out/qd.log 2>&1; grep -E "decide.*cycles|^step" gpurun_out/qd.log | tail -11
