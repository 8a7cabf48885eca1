# full ncu capture (with SASS-level source page) of a few JIT pass kernels of
# the configs[1] circuit; run only after tools/run_cfg1.py exits 0 plain
python tools/run_cfg1.py > gpurun_out/pj_plain.log 2>&1 && \
SVB_JIT_LINEINFO=1 ncu --set full --clock-control none --import-source on -k kpass -s 10 -c 3 \
   -o gpurun_out/prof_jit_cfg1 python tools/run_cfg1.py > gpurun_out/ncu_jit_cfg1.log 2>&1; tail -3 gpurun_out/ncu_jit_cfg1.log
