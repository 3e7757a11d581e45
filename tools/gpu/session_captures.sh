set -x
# full ncu captures at the ranks the bench reaches (after the same command ran clean);
# summarised on the box (the reports with sources are ~36 MB each)
python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/pw15.log 2>&1 || exit 1
tail -2 gpurun_out/pw15.log
cap() {  # pattern name skip steps title
  cmd="ncu --set full --clock-control none --import-source on --nvtx --nvtx-include prof/ -k regex:$1 -c 1 python tools/profile_window.py --skip $3 --steps $4"
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -k "regex:$1" -c 1 -o /tmp/$2 -f python tools/profile_window.py --skip $3 --steps $4 > gpurun_out/$2.log 2>&1
  echo "$2 rc $?"
  python tools/ncu_summary.py /tmp/$2.ncu-rep gpurun_out/$2.md "$5" "$cmd" > gpurun_out/$2.traffic.json
  ncu -i /tmp/$2.ncu-rep --page raw --csv > gpurun_out/$2.raw.csv 2>/dev/null
  rm -f /tmp/$2.ncu-rep
}
cap "k_project_ws" r02_stats_ws_r20 16 2 "r02: statistics pass at r = 20 (k_project_ws<8,3>, a = 512, 4.29 GB increment), bench clocks"
cap "k_syrk_kp" r02_syrk_kp_a168 16 2 "r02: mode-3 raw Gram at a = 168 (k_syrk_kp<21,4,2>, 1.4 GB operand), bench clocks"
cap "k_syrk_kx" r02_syrk_kx_a64 16 2 "r02: mode-2 raw Gram at a = 64 (k_syrk_kx<8>, 4.29 GB increment), bench clocks"
cap "k_project_kc<4" r02_proj64_r21 16 2 "r02: cur3 projection a = 64 -> r = 21 (k_project_kc<4,3,0>), bench clocks"
python tools/profile_window.py --skip 24 --steps 1 > gpurun_out/pw15b.log 2>&1 && \
cap "k_project_ws" r02_stats_ws_r24 24 1 "r02: statistics pass at r = 24 (k_project_ws<8,3>, a = 512), bench clocks"
tail -1 gpurun_out/pw15b.log
python tools/bench_io.py > gpurun_out/r02_io_bench.json 2> gpurun_out/r02_io.err; python -c "
import json; d=json.load(open('gpurun_out/r02_io_bench.json')); print(d['rre']['kernel'])"
