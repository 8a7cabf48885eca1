# full ncu capture (SASS source page) of JIT pass number $1 of configs[1]
python tools/run_cfg1.py > gpurun_out/pj_plain.log 2>&1 && \
SVB_JIT_LINEINFO=1 ncu --set full --clock-control none --import-source on -k kpass -s $1 -c 1 \
   -o gpurun_out/prof_pass$1 python tools/run_cfg1.py > gpurun_out/ncu_pass$1.log 2>&1; tail -1 gpurun_out/ncu_pass$1.log
SVB_PLAN_DEBUG=2 SVB_JIT_DUMP=gpurun_out/jd python -c "
import ctypes, sys
sys.path.insert(0, '.')
from paper_1801_01037_b200 import _lib, workloads
lib=_lib.load(require_cuda=False)
c = workloads.random_layer_circuit(26, 200)
arr,n=_lib.ops_array(c.ops); out=ctypes.c_int()
print(lib.svb_jit_check(26, arr, n, _lib.run_flags(fma=True, jit=True), ctypes.byref(out)))
" 2> gpurun_out/jd_plan.log
