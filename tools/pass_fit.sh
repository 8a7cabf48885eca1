SVB_PLAN_DEBUG=2 python tools/run_cfg1.py > gpurun_out/plan_dbg.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum \
  --clock-control none -k kpass --csv --log-file gpurun_out/pass_fit.csv python tools/run_cfg1.py > gpurun_out/pass_fit.log 2>&1
tail -2 gpurun_out/pass_fit.log
