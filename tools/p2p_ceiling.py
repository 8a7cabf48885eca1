"""Measured NVLink ceiling between GPU pairs (the denominator of the N>1
bench's `frac_of_measured_ceiling`).

    torchrun --nproc-per-node N tools/p2p_ceiling.py [GiB]

Each rank r maps its partner r^1's buffer over CUDA IPC and pulls GiB of it
into local memory, both directions of every pair at once: (a) copy engines
(cudaMemcpyAsync across devices = cudaMemcpyPeerAsync), (b) the SM-driven
k_peer_copy kernel.  CUDA-event timed, slowest rank, best of 3.  Prints one
JSON line on rank 0.  (The same probe runs inside bench.py --gpus N.)"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200.dist import DistEngine, link_ceiling  # noqa: E402


def main():
    gib = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    backend = os.environ.get("SVB_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    world = dist.get_world_size()
    k = world.bit_length() - 1
    nbytes = int(gib * (1 << 30))
    n = max(k + 1, (nbytes // 16).bit_length() - 1 + k)  # slab >= the probe size
    eng = DistEngine(n, peer=True)
    res = link_ceiling(eng, nbytes, "cuda" if backend == "nccl" else "cpu")
    eng.close()
    if dist.get_rank() == 0:
        print(json.dumps({"world": world, "ceiling": res,
                          "nvlink_spec_gbs_per_direction": 900.0}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
