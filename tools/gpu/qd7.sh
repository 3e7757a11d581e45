TTG_TRACE=1 timeout 300 python tools/profile_window.py --skip 24 --steps 2 > gpurun_out/tr.log 2>&1; grep -E "ttg-trace|^step" gpurun_out/tr.log | tail -40
