timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() {
  env $1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep $3 > gpurun_out/$2.json 2> gpurun_out/$2.err
  python -c "import json;d=json.load(open('gpurun_out/$2.json'));r=d['roofline'];print('$2',d['value'],d['e2e']['value'],r['achieved'],r['avg_launch_ms'],r['launches'],d['config']['hbm_passes_per_step'],d['check'])" || tail -5 gpurun_out/$2.err
}
run "X=1" fs5
run "SVB_JIT_FS=4" fs4
run "SVB_JIT_FM=13" fs5fm13
