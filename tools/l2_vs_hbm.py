"""Compute-only vs streaming cost of the specialised passes: the configs[1]
circuit (200 layers) at n = 22 (64 MiB state, L2-resident) and n = 26
(1 GiB, HBM), ns per amplitude per pass, same plan shape (fm 12)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import device, workloads  # noqa: E402

out = {}
for n in [int(x) for x in (sys.argv[1:] or ["22", "23", "24", "26"])]:
    circ = workloads.random_layer_circuit(n, 200)
    st = device.DeviceState.zeros(n)
    device.run_ops(st, circ, fuse=True, fma=True, jit=True)  # compile
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        device.run_ops(st, circ, fuse=True, fma=True, jit=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    passes = device.plan_passes(n, circ, jit=True)
    out[n] = {"ms": ms, "passes": passes, "ns_per_amp_pass": ms * 1e6 / passes / 2 ** n,
              "gate_apps_per_s": len(circ.ops) / ms * 1e3}
    print(n, out[n], flush=True)
print(json.dumps(out))
