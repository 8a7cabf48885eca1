#!/usr/bin/env bash
# per-pass launch times of the configs[1] JIT passes under each tile mode ($MODES)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for m in ${MODES:-2 3}; do
SVB_JIT_MODE=$m python tools/run_cfg1.py > gpurun_out/pj_plain_m$m.log 2>&1 || exit 1
SVB_JIT_MODE=$m timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv \
   -k kpass --log-file gpurun_out/launches_m$m.csv python tools/run_cfg1.py > gpurun_out/ncu_launch_m$m.log 2>&1
done
echo done > gpurun_out/done.txt
