"""Seeded synthetic workloads for the BASELINE.json configs.

There is no public benchmark behind this path; every input is
synthetic, built with numpy's PCG64 ``default_rng(seed)`` so the GPU path and
the CPU reference see identical gate matrices and initial states.

* ``random_unitary2`` / ``random_state_array`` restate the reference test
  fixtures (pkg/tests/conftest.py:24-29, 46-48).
* ``qft_circuit``: config 1 / 4 -- LSB-convention QFT: for j = 0..n-1, H(j)
  then CP(pi/2^(k-j)) control j target k for k > j, then qubit-reversal
  swaps (p, n-1-p) as three CNOTs each.  20 + 190 + 30 = 240 ops at n=20.
* ``random_layer_circuit``: config 2 / 5 -- per layer every qubit q (in
  order) gets one gate uniform over {H,X,Y,Z,S,T,Rx,Ry,Rz}, theta ~
  U[0, 2pi); then n//2 CNOTs on a seeded random perfect matching (permute,
  pair consecutive, control = first).  200 * (26 + 13) = 7,800 ops at n=26.
* ``sweep_ops``: config 3 -- one Haar U per target t = 0..n-1, ``reps``
  applications each, no fusion across reps.
"""

from __future__ import annotations

import math

import numpy as np

from .core import Circuit, Gate2x2, GateOp, phase, rx, ry, rz, standard_gate

SEED_CFG2 = 2026
SEED_CFG3 = 3030
SEED_STATE = 7

LAYER_GATES = ("H", "X", "Y", "Z", "S", "T", "Rx", "Ry", "Rz")


def random_unitary2(rng: np.random.Generator) -> Gate2x2:
    """Haar-ish 2x2 unitary: QR of a complex Gaussian, phase-fixed (conftest.py:24-29)."""
    m = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    q, r = np.linalg.qr(m)
    d = np.diagonal(r)
    return Gate2x2.from_matrix(q * (d / np.abs(d)))


def random_state_array(rng: np.random.Generator, n: int) -> np.ndarray:
    """Normalized complex Gaussian (conftest.py:46-48)."""
    v = rng.normal(size=2**n) + 1j * rng.normal(size=2**n)
    return (v / np.linalg.norm(v)).astype(np.complex128)


def seeded_state(n: int, seed: int) -> np.ndarray:
    """Normalized complex Gaussian that is bit-identical on every host: the
    same PCG64 draws as random_state_array, normalised with an exactly
    rounded sum (math.fsum) instead of BLAS, whose rounding depends on the
    CPU's SIMD width."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=2**n) + 1j * rng.normal(size=2**n)
    s = math.fsum(np.concatenate([v.real * v.real, v.imag * v.imag]).tolist())
    return (v / math.sqrt(s)).astype(np.complex128)


def qft_circuit(n: int) -> Circuit:
    ops = []
    h = standard_gate("H")
    x = standard_gate("X")
    for j in range(n):
        ops.append(GateOp("single", h, j))
        for k in range(j + 1, n):
            ops.append(GateOp("controlled", phase(math.pi / 2 ** (k - j)), k, j))
    for p in range(n // 2):
        a, b = p, n - 1 - p
        ops += [GateOp("controlled", x, b, a), GateOp("controlled", x, a, b),
                GateOp("controlled", x, b, a)]
    return Circuit(n, tuple(ops))


def _layer_gate(name: str, rng: np.random.Generator) -> Gate2x2:
    if name in ("Rx", "Ry", "Rz"):
        theta = float(rng.uniform(0.0, 2.0 * math.pi))
        return {"Rx": rx, "Ry": ry, "Rz": rz}[name](theta)
    return standard_gate(name)


def random_layer_circuit(n: int, layers: int, seed: int = SEED_CFG2) -> Circuit:
    rng = np.random.default_rng(seed)
    x = standard_gate("X")
    ops = []
    for _ in range(layers):
        for q in range(n):
            name = LAYER_GATES[int(rng.integers(len(LAYER_GATES)))]
            ops.append(GateOp("single", _layer_gate(name, rng), q))
        perm = rng.permutation(n)
        for i in range(0, n - 1, 2):
            c, t = int(perm[i]), int(perm[i + 1])
            ops.append(GateOp("controlled", x, t, c))
    return Circuit(n, tuple(ops))


def sweep_ops(n: int, reps: int = 10, seed: int = SEED_CFG3) -> Circuit:
    rng = np.random.default_rng(seed)
    ops = []
    for t in range(n):
        g = random_unitary2(rng)
        ops += [GateOp("single", g, t)] * reps
    return Circuit(n, tuple(ops))


def oracle_ops(circuit: Circuit):
    """(gate, target, control|None) triples, the form oracle/ consumes."""
    return [(op.gate, op.target, op.control) for op in circuit.ops]


def inverse_circuit(circuit: Circuit) -> Circuit:
    """U^dagger of a circuit: ops reversed, every gate conjugate-transposed
    (round-trip checks at sizes no CPU oracle holds)."""
    ops = []
    for op in reversed(circuit.ops):
        g = op.gate
        gi = Gate2x2(complex(g.q11).conjugate(), complex(g.q21).conjugate(),
                     complex(g.q12).conjugate(), complex(g.q22).conjugate())
        ops.append(GateOp(op.kind, gi, op.target, op.control))
    return Circuit(circuit.n, tuple(ops))


def bit_reverse(x: int, n: int) -> int:
    return int(format(x, f"0{n}b")[::-1], 2)


def qft_basis_amplitude(x: int, y: int, n: int) -> complex:
    """<y| qft_circuit(n) |x> = exp(2 pi i br(x) br(y) / 2^n) / 2^(n/2) (SURVEY
    8(c) known answer for the LSB-convention QFT with final reversal swaps);
    the phase is reduced exactly in integers, so it holds at n = 33/34 where
    br(x) br(y) overflows int64.  A closed form used as a size-independent
    check in bench.py's multi-GPU line (the tests check it against the
    oracle's own copy)."""
    N = 1 << n
    ph = (bit_reverse(x, n) * bit_reverse(y, n)) % N
    return complex(np.exp(2j * np.pi * ph / N) / np.sqrt(N))
