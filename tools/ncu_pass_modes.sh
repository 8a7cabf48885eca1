#!/usr/bin/env bash
# full ncu (SASS source page) of configs[1] JIT pass $PASS under each tile mode ($MODES)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for m in ${MODES:-2 3}; do
SVB_JIT_MODE=$m python tools/run_cfg1.py > gpurun_out/pj_plain_m$m.log 2>&1 || exit 1
SVB_JIT_MODE=$m SVB_JIT_LINEINFO=1 timeout 900 ncu --set full --clock-control none --import-source on -k kpass -s ${PASS:-2} -c 1 \
   -o gpurun_out/prof_p${PASS:-2}_m$m python tools/run_cfg1.py > gpurun_out/ncu_p_m$m.log 2>&1; tail -1 gpurun_out/ncu_p_m$m.log
done
echo done > gpurun_out/done.txt
