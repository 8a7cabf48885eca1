#!/usr/bin/env bash
# full round check: GPU tests, smoke, full bench, reference arm, launch list of
# the bench command, one full ncu capture of a kpass launch
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rA --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-sweep --no-cold --no-seam > gpurun_out/ncu_launch_bench.log 2>&1
SVB_JIT_LINEINFO=1 timeout 900 ncu --set full --clock-control none --import-source on -k kpass -s 60 -c 1 \
   -o gpurun_out/prof_kpass_r02 python tools/run_cfg1.py > gpurun_out/ncu_kpass_r02.log 2>&1
echo done > gpurun_out/done.txt
