"""Per-step wall time and JIT activity of DistEngine.run over repeated runs of
one circuit (the layout persists across runs, so a run's local segments are
new circuits in physical qubits until the layout cycle closes).

    SVB_DIST_BACKEND=gloo torchrun --nproc-per-node 2 tools/dist_steps.py qft 26 10
"""
import ctypes
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import _lib, workloads  # noqa: E402
from paper_1801_01037_b200.dist import DistEngine, device_gaussian  # noqa: E402

kind, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
backend = os.environ.get("SVB_DIST_BACKEND", "nccl")
local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
torch.cuda.set_device(local)
dist.init_process_group(backend) if backend != "nccl" else dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = "cuda" if backend == "nccl" else "cpu"
circ = workloads.qft_circuit(n) if kind == "qft" else workloads.random_layer_circuit(n, 50)
eng = DistEngine(n, fma=True, jit=True, layout=True, peer=True)
device_gaussian(eng, 7, dev)
lib = _lib.load()


def counters():
    a, b = ctypes.c_long(), ctypes.c_long()
    lib.svb_jit_counters(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


for s in range(steps):
    c0 = counters()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run(circ)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    c1 = counters()
    if dist.get_rank() == 0:
        print(f"step {s}: {dt * 1e3:9.1f} ms   jit counters (disk hits, compiles) +{c1[0] - c0[0]} +{c1[1] - c0[1]}", flush=True)
eng.close()
dist.barrier()
dist.destroy_process_group()
