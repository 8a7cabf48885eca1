python tools/prof_gates.py 26 jit > gpurun_out/pj_plain.log 2>&1 && \
SVB_JIT_LINEINFO=1 ncu --set full --clock-control none --import-source on -k kpass -s 1 -c 1 -o gpurun_out/prof_jit_src python tools/prof_gates.py 26 jit > gpurun_out/ncu_jit_src.log 2>&1; tail -3 gpurun_out/ncu_jit_src.log
