"""Short driver for ncu captures: a few launches of each gate kernel class at
n=28 (4 GiB state, well beyond L2).  Run plain first, then under ncu.

    python tools/prof_gates.py [n] [fused|jit]
      (default)  single-gate kernels, then one fused random-layer run
      fused      only the fused run, interpreter kernel (k_fused)
      jit        only the fused run, NVRTC-specialised kernels (kpass)
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import device, standard_gate, workloads, phase  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
mode = sys.argv[2] if len(sys.argv) > 2 else ""
st = device.DeviceState.random(n, seed=1)
u = workloads.random_unitary2(__import__("numpy").random.default_rng(1))
if mode not in ("fused", "jit"):
    for t in (0, 3, 10, n - 1):
        device.apply_single(st, u, t)            # k_pair_low / k_pair_high, general
        device.apply_single(st, standard_gate("h"), t)
    device.apply_controlled(st, standard_gate("x"), 2, 20)
    device.apply_single(st, standard_gate("t"), 7)   # k_diag, half the state
    device.apply_controlled(st, phase(0.3), 5, 9)    # k_diag, quarter
circ = workloads.random_layer_circuit(n, 2, seed=3)
device.run_ops(st, circ, fuse=True, fma=True, jit=(mode == "jit"))
torch.cuda.synchronize()
print("norm", device.norm2(st))
