"""BASELINE configs[3] shape on ONE B200: QFT on n=33 qubits (2^33 amplitudes,
128 GiB of HBM), checked by known answers and a round trip.

* fused single-rank run (svb_run_ops) from a basis state |x>: sampled output
  amplitudes vs the closed form exp(2 pi i br(x) br(y) / N) / sqrt(N);
* the same circuit through the partitioned engine with 2^k emulated ranks
  (k global qubits; every H / CP on them goes through the peer-memory pair
  kernel), then the inverse circuit: back to |x> within 1e-12.

Usage: python tools/scale_qft33.py [n] [k]   (n=33, k=3 default)
Writes one JSON line.  Not part of bench.py (about a minute of GPU time).
"""

import json
import math
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402  (checker: closed-form known answers)
from paper_1801_01037_b200 import Circuit, GateOp, PartitionPlan, SCHEME_B, device, engine, workloads  # noqa: E402


def inverse(circ: Circuit) -> Circuit:
    ops = []
    for op in reversed(circ.ops):
        g = op.gate
        gi = type(g)(complex(g.q11).conjugate(), complex(g.q21).conjugate(),
                     complex(g.q12).conjugate(), complex(g.q22).conjugate())
        ops.append(GateOp(op.kind, gi, op.target, op.control))
    return Circuit(circ.n, tuple(ops))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    N = 1 << n
    x = 0x1234567 % N
    circ = workloads.qft_circuit(n)
    rng = np.random.default_rng(5)
    ys = [0, 1, N - 1] + [int(v) for v in rng.integers(0, N, size=29)]
    out = {"n": n, "k": k, "ops": len(circ.ops), "x": x}

    # fused, one rank
    st = device.DeviceState.zeros(n)
    st.amps.zero_()
    st.amps[x] = 1.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    device.run_ops(st, circ)
    torch.cuda.synchronize()
    out["fused_s"] = time.perf_counter() - t0
    out["fused_passes"] = device.plan_passes(n, circ)
    got = st.amps[torch.tensor(ys, device="cuda")].cpu().numpy()
    want = np.array([oracle.qft_basis_amplitude(x, y, n) for y in ys])
    out["fused_known_answer_maxerr"] = float(np.max(np.abs(got - want)))
    out["fused_norm"] = device.norm2(st)

    # the bench's fast path (FMA + NVRTC-specialised 12-qubit passes): once to
    # plan and compile, then timed
    for rep in range(2):
        st.amps.zero_()
        st.amps[x] = 1.0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        device.run_ops(st, circ, fma=True, jit=True)
        torch.cuda.synchronize()
        out["fast_first_s" if rep == 0 else "fast_s"] = time.perf_counter() - t0
    out["fast_passes"] = device.plan_passes(n, circ, jit=True)
    got = st.amps[torch.tensor(ys, device="cuda")].cpu().numpy()
    out["fast_known_answer_maxerr"] = float(np.max(np.abs(got - want)))
    out["fast_norm"] = device.norm2(st)
    del st
    torch.cuda.empty_cache()

    # partitioned engine, 2^k emulated ranks on this GPU, then the inverse
    plan = PartitionPlan(n, k)
    ds = engine.dist_init(plan, scheme=SCHEME_B)
    L = plan.local_len
    for s in ds.slabs:
        s.zero_()
    ds.slabs[x // L][x % L] = 1.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    # op by op on the existing slabs (run_circuit would allocate a second state)
    for op in circ.ops:
        if op.kind == "single":
            if op.target < n - k:
                engine.dist_apply_local(ds, op.gate, op.target)
            else:
                engine.dist_apply_scheme_b(ds, op.gate, op.target)
        else:
            engine.dist_apply_controlled(ds, op.gate, op.control, op.target)
    ds.sync()
    out["engine_s"] = time.perf_counter() - t0
    got = np.array([complex(ds.slabs[y // L][y % L].item()) for y in ys])
    out["engine_known_answer_maxerr"] = float(np.max(np.abs(got - want)))
    out["engine_peer_bytes_per_rank"] = ds.peer_bytes()[0]
    t0 = time.perf_counter()
    for op in inverse(circ).ops:
        if op.kind == "single":
            if op.target < n - k:
                engine.dist_apply_local(ds, op.gate, op.target)
            else:
                engine.dist_apply_scheme_b(ds, op.gate, op.target)
        else:
            engine.dist_apply_controlled(ds, op.gate, op.control, op.target)
    ds.sync()
    out["engine_inverse_s"] = time.perf_counter() - t0
    peak = complex(ds.slabs[x // L][x % L].item())
    out["round_trip_abs_err_at_x"] = abs(peak - 1.0)
    out["round_trip_norm"] = engine.dist_norm2(ds)
    out["round_trip_residual"] = math.sqrt(max(0.0, out["round_trip_norm"] - abs(peak) ** 2))
    ds.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
