set -x
python tools/profile_window.py --skip 17 --steps 1 > gpurun_out/pw12.log 2>&1 && \
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_decide -s 6 -c 1 -o gpurun_out/r02_decide_full -f python tools/profile_window.py --skip 17 --steps 1 > gpurun_out/ncu12.log 2>&1
echo "rc $?"; tail -3 gpurun_out/ncu12.log
