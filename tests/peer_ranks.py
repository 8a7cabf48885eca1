"""Ranks of the peer-memory transport test (tests/test_gpu_peer.py): torchrun
starts WORLD_SIZE processes that all use cuda:0 (CUDA IPC works between
processes on one device) with a gloo control plane; each runs DistEngine
with peer=True -- exchanges and layout swaps as kernels reading and writing
the partner's slab -- and rank 0 checks the gathered state against the
oracle.  Exit status 0 = every check passed."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
from paper_1801_01037_b200 import Circuit, GateOp, phase, standard_gate, workloads as w  # noqa: E402
from paper_1801_01037_b200.dist import DistEngine  # noqa: E402

dist.init_process_group("gloo")
torch.cuda.set_device(0)
rank, world = dist.get_rank(), dist.get_world_size()
n = 14
k = world.bit_length() - 1
rng = np.random.default_rng(7)
x, h = standard_gate("x"), standard_gate("h")
pool = [x, h, standard_gate("t"), phase(0.7), w.random_unitary2(rng), w.random_unitary2(rng)]
ops = []
for _ in range(160):
    g = pool[int(rng.integers(len(pool)))]
    t = int(rng.integers(n - k, n)) if rng.random() < 0.4 else int(rng.integers(n))  # global targets often
    if rng.random() < 0.5:
        c = int(rng.integers(n))
        while c == t:
            c = int(rng.integers(n))
        ops.append(GateOp("controlled", g, t, c))
    else:
        ops.append(GateOp("single", g, t))
circ = Circuit(n, tuple(ops))
a = w.random_state_array(np.random.default_rng(8), n)
want = oracle.run_ops(a.copy(), w.oracle_ops(circ)) if rank == 0 else None
want2 = oracle.run_ops(want.copy(), w.oracle_ops(circ)) if rank == 0 else None  # the circuit twice
bad = 0
# device-side pairwise sync (default) for every layout x arithmetic mode, and
# the host-barrier fallback for two of them
cases = [(layout, fma, True) for layout in (False, True) for fma in (False, True)]
cases += [(False, False, False), (True, True, False)]
for layout, fma, gpu_sync in cases:
    eng = DistEngine(n, initial=a, peer=True, layout=layout, fma=fma, jit=fma, gpu_sync=gpu_sync)
    assert eng.peer and eng.gpu_sync == gpu_sync, "peer transport / device sync unavailable"
    eng.run(circ)
    eng.run(circ)  # twice: the flag counts keep matching across runs
    out = eng.gather()
    st = eng.stats
    eng.close()
    if rank == 0:
        err = float(np.max(np.abs(out - want2)))
        ok = err <= 1e-12 and (st.exchanges + st.swaps) > 0
        print(f"world {world} layout {layout} fma {fma} gpu_sync {gpu_sync}: max err {err:.2e}, "
              f"exchanges {st.exchanges}, swaps {st.swaps} {'ok' if ok else 'FAIL'}", flush=True)
        bad += not ok
dist.barrier()
dist.destroy_process_group()
sys.exit(1 if bad else 0)
