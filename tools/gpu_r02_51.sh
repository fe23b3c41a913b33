export PATH=/usr/local/cuda/bin:$PATH
for c in c4 c5; do
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__grid_size,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio --clock-control none -k regex:"p2_near|p2_proxy|half2" -c 3 python tools/ncu_step.py --config $c --matvecs 1 2>&1 | grep -E "p2_near|p2_proxy|half2|duration|fp64|issue_active|inst_executed|grid_size|stalled" 
done > gpurun_out/r02_near_c4c5_ncu.log 2>&1
cat gpurun_out/r02_near_c4c5_ncu.log
