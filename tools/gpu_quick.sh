#!/usr/bin/env bash
# one gpurun call: selected GPU tests ($TESTS) + bench ($BENCH_ARGS)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ "${TESTS:-}" != "none" ]; then
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -rA -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [ -n "${BENCH_ARGS:-}" ]; then
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
fi
echo done > gpurun_out/done.txt
