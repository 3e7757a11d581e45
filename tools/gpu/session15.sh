set -x
# full ncu captures at the ranks the bench reaches (after the same command ran clean)
python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/pw15.log 2>&1 || exit 1
tail -2 gpurun_out/pw15.log
for spec in "k_project_ws:r02_stats_ws_r20" "k_syrk_kp:r02_syrk_kp_a168" "k_syrk_kx:r02_syrk_kx_a64" "k_project_kc<4:r02_proj64_r21"; do
  pat=${spec%%:*}; name=${spec##*:}
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -k "regex:$pat" -c 1 -o gpurun_out/$name -f python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/$name.log 2>&1
  echo "$name rc $?"
done
python tools/profile_window.py --skip 24 --steps 1 > gpurun_out/pw15b.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -k "regex:k_project_ws|k_project_kc<8, 3" -c 1 -o gpurun_out/r02_stats_r24 -f python tools/profile_window.py --skip 24 --steps 1 > gpurun_out/r02_stats_r24.log 2>&1
echo "r24 rc $?"; tail -2 gpurun_out/pw15b.log
