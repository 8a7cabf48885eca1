import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np
import oracle
from paper_1801_01037_b200 import device, workloads as w, Circuit
n, L, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
circ = w.random_layer_circuit(n, L, seed=seed)
a = w.random_state_array(np.random.default_rng(77), n)
want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=16)
got = device.simulate(circ, a.copy(), fma=True, jit=True)
print(sys.argv[1:], {k: v for k, v in os.environ.items() if k.startswith("SVB_")}, np.max(np.abs(got - want)), flush=True)
