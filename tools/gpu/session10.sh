set -x
for i in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export TTG_SPEC_FAKE=1; else unset TTG_SPEC_FAKE; fi
  python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SPEC_FAKE=$v', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][-6:])"
done
done
unset TTG_SPEC_FAKE
TTG_DEBUG=1 timeout 300 python tools/profile_window.py --skip 17 --steps 1 > gpurun_out/r02_pw_debug.log 2>&1; grep "eig_top" gpurun_out/r02_pw_debug.log | tail -8
