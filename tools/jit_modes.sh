# JIT parity + configs[1] bench variants: "mode ctas flow tag"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
run() {
  SVB_JIT_MODE=$1 SVB_JIT_CTAS=$2 SVB_FUSE_FLOW=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep $5 > gpurun_out/$4.json 2> gpurun_out/$4.err
  python -c "import json;d=json.load(open('gpurun_out/$4.json'));r=d['roofline'];print('$4',d['value'],d['e2e']['value'],r['achieved'],r['avg_launch_ms'],r['launches'])" || tail -5 gpurun_out/$4.err
}
run 0 4 3 c4
run 0 4 3 c4interp --no-jit
bash tools/pass_fit.sh
