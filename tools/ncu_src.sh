#!/usr/bin/env bash
# launch list of the configs[1] JIT passes + full ncu (SASS source page) of passes $PASSES
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python tools/run_cfg1.py > gpurun_out/pj_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   -k kpass --log-file gpurun_out/launches_cfg1.csv python tools/run_cfg1.py > gpurun_out/ncu_launch.log 2>&1
for p in ${PASSES:-50}; do
SVB_JIT_LINEINFO=1 timeout 900 ncu --set full --clock-control none --import-source on -k kpass -s $p -c 1 \
   -o gpurun_out/prof_pass$p python tools/run_cfg1.py > gpurun_out/ncu_pass$p.log 2>&1; tail -1 gpurun_out/ncu_pass$p.log
done
echo done > gpurun_out/done.txt
