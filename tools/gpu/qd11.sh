ALGO=ice K0=10 TTG_NO_SPEC=1 TTG_DEBUG=1 python tools/probe/cfg1_window.py > gpurun_out/c1d.log 2>&1; grep -E "decide a=|eig_top|eig a=|^1[01] " gpurun_out/c1d.log | tail -40
