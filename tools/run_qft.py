"""One JIT run of the QFT at n qubits on one GPU from a seeded device state -- a
short driver for ncu launch lists / captures of configs[3]'s passes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import device, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
circ = workloads.qft_circuit(n)
st = device.DeviceState.zeros(n)
st.amps[12345] = 1.0
st.amps[0] = 0.0
for _ in range(2):
    device.run_ops(st, circ, fuse=True, fma=True, jit=True)
torch.cuda.synchronize()
print("norm", device.norm2(st))
