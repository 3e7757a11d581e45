# full ncu captures of the two new latency-bound kernels (summarised on the box)
set -x
python tools/profile_window.py --skip 16 --steps 2 > gpurun_out/pw15.log 2>&1 || exit 1
cap() {
  cmd="ncu --set full --clock-control none --import-source on --nvtx --nvtx-include prof/ -k regex:$1 -s $6 -c 1 python tools/profile_window.py --skip $3 --steps $4"
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "prof/" -k "regex:$1" -s $6 -c 1 -o /tmp/$2 -f python tools/profile_window.py --skip $3 --steps $4 > gpurun_out/$2.log 2>&1
  echo "$2 rc $?"
  python tools/ncu_summary.py /tmp/$2.ncu-rep gpurun_out/$2.md "$5" "$cmd" > gpurun_out/$2.traffic.json
  rm -f /tmp/$2.ncu-rep
}
cap "k_decide" r02_decide_a168 16 2 "r02: k_decide<2> at a = 168, r_old = 20 (mode 3 of the update step; one CTA)" 0
cap "k_project_tail" r02_project_tail 16 2 "r02: k_project_tail (modes 5-7 of the statistics chain, 256 CTAs)" 0
