# ncu of one bnreg_best_subsets call (its 3 passes) at cfg5; then the timing run without ncu
timeout 600 python tools/bps_time.py 5 > gpurun_out/bps_time5.log 2>&1
timeout 600 python tools/bps_time.py 4 >> gpurun_out/bps_time5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem --clock-control none -k regex:bps_ -c 3 --csv python tools/bps_time.py 5 > gpurun_out/bps_ncu.csv 2> gpurun_out/bps_ncu.err; tail -3 gpurun_out/bps_ncu.err
cat gpurun_out/bps_time5.log
