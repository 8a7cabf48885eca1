"""One run of a gate-heavy one-kind circuit (tools/gate_cost.py shape) for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import Circuit, GateOp, device, rx, standard_gate  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "h"
n, q, G = 26, 12, 1500
rng = np.random.default_rng(5)
mk = (lambda: rx(float(rng.uniform(0, 6.28)))) if kind == "rx" else (lambda: standard_gate(kind))
circ = Circuit(n, tuple(GateOp("single", mk(), i % q) for i in range(G)))
st = device.DeviceState.zeros(n)
device.run_ops(st, circ, fma=True, jit=True)
torch.cuda.synchronize()
print("ok")
