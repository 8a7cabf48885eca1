"""Per-gate-type cost inside specialised passes: circuits of one gate kind on
qubits 0..q-1 (so passes are gate-heavy), n = 26; time per pass and per gate
application beyond an empty (gate-free) pass."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_01037_b200 import Circuit, GateOp, device, phase, rx, ry, rz, standard_gate  # noqa: E402

n = 26
rng = np.random.default_rng(5)


def timed(circ, reps=3):
    st = device.DeviceState.zeros(n)
    device.run_ops(st, circ, fma=True, jit=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        device.run_ops(st, circ, fma=True, jit=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


kinds = {
    "H": lambda: standard_gate("h"), "X": lambda: standard_gate("x"), "Y": lambda: standard_gate("y"),
    "Z": lambda: standard_gate("z"), "S": lambda: standard_gate("s"), "T": lambda: standard_gate("t"),
    "Rx": lambda: rx(float(rng.uniform(0, 6.28))), "Ry": lambda: ry(float(rng.uniform(0, 6.28))),
    "Rz": lambda: rz(float(rng.uniform(0, 6.28))),
}
out = {}
q = 12
G = 1500
for name, mk in list(kinds.items()) + [("CNOT", None), ("CP", None)]:
    ops = []
    for i in range(G):
        if name == "CNOT":
            c, t = rng.choice(q, size=2, replace=False)
            ops.append(GateOp("controlled", standard_gate("x"), int(t), int(c)))
        elif name == "CP":
            c, t = rng.choice(q, size=2, replace=False)
            ops.append(GateOp("controlled", phase(float(rng.uniform(0, 6.28))), int(t), int(c)))
        else:
            ops.append(GateOp("single", mk(), i % q))
    circ = Circuit(n, tuple(ops))
    passes = device.plan_passes(n, circ, jit=True)
    ms = timed(circ)
    out[name] = {"ms": round(ms, 3), "passes": passes, "us_per_pass": round(ms * 1e3 / passes, 1),
                 "us_per_gate": round(ms * 1e3 / G, 3)}
    print(name, out[name], flush=True)
print(json.dumps(out))
