# A/B on one box: tools/ab.sh <libA> <libB> [rounds]  (alternating bench runs)
A=$1; B=$2; N=${3:-3}
for i in $(seq 1 $N); do
  for L in $A $B; do
    TTG_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-clocks > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['value'],1), [round(s['device_ms'],2) for s in d['steps_detail']][:4])"
  done
done
