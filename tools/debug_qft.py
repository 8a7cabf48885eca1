"""Find the first op where the GPU diverges from the oracle (debug aid)."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
from paper_1801_01037_b200 import device, workloads as w  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
a = w.random_state_array(np.random.default_rng(w.SEED_STATE), n)
circ = w.qft_circuit(n)
ref = a.copy()
st = device.DeviceState.from_host(a)
for i, op in enumerate(circ.ops):
    oracle.run_ops(ref, [(op.gate, op.target, op.control)])
    if op.control is None:
        device.apply_single(st, op.gate, op.target)
    else:
        device.apply_controlled(st, op.gate, op.control, op.target)
    got = st.to_host().amps
    if not np.array_equal(got, ref):
        d = np.nonzero(got != ref)[0]
        print(f"op {i}: t={op.target} c={op.control} gate={op.gate} ndiff={d.size} first={d[:8]}")
        j = d[0]
        print("  got", got[j], "want", ref[j], "maxerr", np.max(np.abs(got - ref)))
        st = device.DeviceState.from_host(ref)  # resync and continue
        if i > 200:
            break
print("done")
out = device.simulate(circ, a.copy(), fuse=False)
ref2 = oracle.run_ops(a.copy(), w.oracle_ops(circ))
print("simulate vs oracle equal:", np.array_equal(out, ref2), np.max(np.abs(out - ref2)))
