"""Host-only numerics of the runtime-specialised passes: the CUDA C that the
JIT generates for a circuit (SVB_JIT_DUMP) is compiled as C++ and run over
a numpy state by tools/jit_emu.py (one std::thread per CUDA thread, a
barrier per __syncthreads), then compared with the oracle.  This checks the
generator -- tile-uniform predicates, pending swaps, per-thread phases,
unit folding, factor extraction, layout rotation -- without a GPU; the GPU
tests check the same circuits on the device."""

import ctypes
import os
import shutil
import sys

import numpy as np
import pytest

import oracle
from paper_1801_01037_b200 import Circuit, GateOp, _lib, device, standard_gate, workloads as w

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import jit_emu  # noqa: E402

TOL = 1e-12


def _controlled_heavy(n, rng, count):
    x = standard_gate("x")
    pool = [standard_gate(g) for g in "XYZHST"] + [x, x, w.random_unitary2(rng), w.random_unitary2(rng)]
    ops = []
    for _ in range(count):
        g = pool[int(rng.integers(len(pool)))]
        if rng.random() < 0.6:
            c, t = rng.choice(n, size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
        else:
            ops.append(GateOp("single", g, int(rng.integers(n))))
    return Circuit(n, tuple(ops))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
@pytest.mark.parametrize("case,n,fm", [("layers", 15, 11), ("qft", 15, 11), ("controlled", 15, 11),
                                       ("layers", 17, 12), ("controlled", 17, 12), ("qft", 17, 12)])
def test_generated_passes_match_oracle(case, n, fm, tmp_path, monkeypatch):
    # fm 11: one shared buffer, 4 CTAs/SM; fm 12: next-tile prefetch (mode 2)
    monkeypatch.setenv("SVB_JIT_FM", str(fm))
    rng = np.random.default_rng(31)
    circ = {"layers": lambda: w.random_layer_circuit(n, 8, seed=5),
            "qft": lambda: w.qft_circuit(n),
            "controlled": lambda: _controlled_heavy(n, rng, 160)}[case]()
    lib = _lib.load(require_cuda=False)
    monkeypatch.setenv("SVB_JIT_DUMP", str(tmp_path))
    arr, nops = _lib.ops_array(circ.ops)
    out = ctypes.c_int()
    rc = lib.svb_jit_check(n, arr, nops, _lib.run_flags(fma=True), ctypes.byref(out))
    if rc == _lib.SVB_ESTATE and b"NVRTC not available" in lib.svb_last_error():
        pytest.skip("NVRTC not available")
    assert rc == 0, lib.svb_last_error()
    monkeypatch.delenv("SVB_JIT_DUMP")
    # every step of the plan must be a fused pass for the emulation to be the
    # whole circuit
    # a trailing SWAP network (the QFT's reversal) is not part of the generated
    # passes: svb_run_ops applies it with k_swap_bits in one pass of its own
    tail = lib.svb_swap_suffix(n, arr, nops)
    steps = device.plan_passes(n, circ, jit=True) - (1 if tail else 0)
    npass = len([f for f in os.listdir(tmp_path) if f.endswith(".cu")])
    if steps != npass:
        pytest.skip(f"plan has single-gate steps ({steps} steps, {npass} passes)")
    a = w.random_state_array(rng, n)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=4)
    got = jit_emu.run_passes(str(tmp_path), a.copy(), grid=3)[-1]  # several tiles per CTA
    if tail:
        got = oracle.run_ops(got, w.oracle_ops(Circuit(n, circ.ops[nops - tail:])), workers=4)
    assert np.max(np.abs(got - want)) <= TOL
