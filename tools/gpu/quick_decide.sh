TTG_DEBUG=1 timeout 300 python tools/profile_window.py --skip 17 --steps 1 > gpurun_out/qd.log 2>&1; grep -E "decide|eig_top|^step" gpurun_out/qd.log | tail -14
for v in 1 0; do
  if [ $v = 1 ]; then export TTG_NO_DECIDE=1; else unset TTG_NO_DECIDE; fi
  python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NO_DECIDE=$v', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
done
unset TTG_NO_DECIDE
timeout 600 ncu --nvtx --nvtx-include "prof/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_pw_launches2.csv python tools/profile_window.py --skip 17 --steps 1 > gpurun_out/r02_pw_ncu2.log 2>&1; echo "ncu rc $?"
