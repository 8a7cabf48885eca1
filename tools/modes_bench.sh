#!/usr/bin/env bash
# configs[1] bench (kernel-only) under each JIT tile mode ($MODES), plus per-pass ncu launch lists
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for m in ${MODES:-2 4}; do
SVB_JIT_MODE=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep --no-cold --no-seam > gpurun_out/bench_m$m.json 2> gpurun_out/bench_m$m.err
done
if [ -n "${NCU:-}" ]; then MODES="${MODES:-2 4}" bash tools/ncu_modes.sh; fi
echo done > gpurun_out/done.txt
