SVB_PLAN_DEBUG=3 python -c "import sys; sys.path.insert(0, '.'); from paper_1801_01037_b200 import device, workloads; device.plan_stats(26, workloads.random_layer_circuit(26, 200), jit=True)" > gpurun_out/plan_dbg.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum \
  --clock-control none -k kpass --csv --log-file gpurun_out/pass_fit.csv python tools/run_cfg1.py > gpurun_out/pass_fit.log 2>&1
tail -2 gpurun_out/pass_fit.log
