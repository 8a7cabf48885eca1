# configs[1] bench across JIT variants: "env tag"
run() {
  env $1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-sweep > gpurun_out/$2.json 2> gpurun_out/$2.err
  python -c "import json;d=json.load(open('gpurun_out/$2.json'));r=d['roofline'];print('$2',d['value'],d['e2e']['value'],r['achieved'],r['avg_launch_ms'],r['launches'])" || tail -5 gpurun_out/$2.err
}
run "SVB_FUSE_PLANNER=2 SVB_FUSE_COMMUTE=0" la
run "SVB_FUSE_PLANNER=3 SVB_FUSE_COMMUTE=1" beam
run "SVB_FUSE_PLANNER=3 SVB_FUSE_COMMUTE=0" beamnc
run "SVB_FUSE_PLANNER=3 SVB_BEAM_D=3" beam3
