"""Where does a fused pass spend its time: arithmetic or HBM?

Runs the configs[1] random-layer circuit (200 layers) through the JIT pass
kernels at several n and reports the average pass time per 2^26 amplitudes.
At n <= 22 the state (64 MiB) stays in the 126 MB L2, so the time is the
kernel's arithmetic/issue bound; at n = 26 (1 GiB) it is the real pass.

    python tools/pass_split.py [--interp]
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import _lib, device, workloads  # noqa: E402

jit = "--interp" not in sys.argv
for n in (20, 22, 24, 26):
    circ = workloads.random_layer_circuit(n, 200)
    st = device.DeviceState.zeros(n)
    for _ in range(2):
        device.run_ops(st, circ, fuse=True, fma=True, jit=jit)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    device.run_ops(st, circ, fuse=True, fma=True, jit=jit)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    name = "kpass_jit" if jit else "k_fused"
    launches, ms, _ = prof[name]
    per = ms / launches
    scale = 2.0 ** (26 - n)
    print(f"n={n:2d} passes={launches:4d} avg pass {per * 1e3:8.1f} us  "
          f"-> per 2^26 amps {per * scale * 1e3:8.1f} us  ({2 * 16 * 2**n / (per * 1e-3) / 1e9:7.1f} GB/s)")
