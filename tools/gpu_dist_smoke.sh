#!/usr/bin/env bash
# N>1 bench path on ONE GPU: 2 ranks share cuda:0 over a gloo control plane
# (functional smoke at reduced n; its timings are not a multi-GPU number)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q -x > gpurun_out/pytest_peer.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_peer.log
SVB_DIST_BACKEND=gloo SVB_BENCH_QFT_N=${QN:-26} SVB_BENCH_CFG4=1 SVB_BENCH_CFG4_N=${QN:-26} timeout 900 \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 \
  bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_dist2.json 2> gpurun_out/bench_dist2.err
echo "rc=$?" >> gpurun_out/bench_dist2.err
echo done > gpurun_out/done.txt
