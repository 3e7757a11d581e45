python tools/bench_io.py > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:k_rre_partial -c 1 -o /tmp/rre -f python tools/bench_io.py > gpurun_out/rre_ncu.log 2>&1
python tools/ncu_summary.py /tmp/rre.ncu-rep gpurun_out/r02_rre_full.md "r02: k_rre_partial<16> (cfg3, 64 observations, r = 14)" "ncu --set full --clock-control none -k regex:k_rre_partial -c 1 python tools/bench_io.py"
ncu -i /tmp/rre.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for k,val in zip(h,v):
    if any(s in k for s in ['smsp__average_warps_issue_stalled','sm__warps_active.avg.pct','smsp__issue_active.avg.pct','l1tex__t_sector_hit_rate','sm__inst_executed_pipe_lsu','smsp__inst_executed_pipe_fp64','dram__throughput','gpu__time_duration']): print(k,val)
" > gpurun_out/rre_stalls.txt
