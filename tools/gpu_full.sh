# full round check: GPU tests, smoke, full bench (+ reference arm), launch list, ncu of kpass
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep > gpurun_out/ncu_launch.log 2>&1
bash tools/ncu_jit.sh
