export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python tools/build_probe.py --config c3 --builds 3 > gpurun_out/r02_build_c3.log 2>&1
timeout 300 python tools/build_probe.py --config c4 --builds 2 > gpurun_out/r02_build_c4.log 2>&1
cat gpurun_out/r02_build_c3.log gpurun_out/r02_build_c4.log
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warp_latency_issue_stalled_barrier.ratio
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:aca_kernel -c 8 --csv --log-file gpurun_out/r02_c3_aca_metrics.csv python tools/ncu_step.py --config c3 --matvecs 0 > gpurun_out/r02_c3_aca_metrics.log 2>&1
tail -3 gpurun_out/r02_c3_aca_metrics.log
