# N=1 bench with / without the in-library launch profiler, twice each
for i in 1 2; do
python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('prof',d['value'],d['ms_per_step'],d['clocks'])"
SVB_BENCH_NOPROF=1 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('noprof',d['value'],d['ms_per_step'],d['clocks'])"
done
