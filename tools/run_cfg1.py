"""One JIT run of the configs[1] circuit (n=26, 200 layers) -- a short
driver for ncu launch lists and SVB_PLAN_DEBUG plan dumps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import device, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
circ = workloads.random_layer_circuit(n, 200)
st = device.DeviceState.zeros(n)
device.run_ops(st, circ, fuse=True, fma=True, jit=True)
torch.cuda.synchronize()
print("norm", device.norm2(st))
