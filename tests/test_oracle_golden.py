"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz,
produced by tests/golden/make_golden.py importing svsim)."""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import circuit_from_rows, gate_from_q, golden, split_cases
from paper_1801_01037_b200 import workloads as w


def canon_sha(a):
    v = np.ascontiguousarray(a, dtype=np.complex128).view(np.float64) + 0.0
    return hashlib.sha256(v.tobytes()).hexdigest()


@pytest.mark.parametrize("workers", [1, 4])
def test_oracle_single_bit_exact_vs_reference(workers):
    z = golden("kernel_single.npz")
    ins = split_cases(z["meta"][:, 0], z["inp"])
    outs = split_cases(z["meta"][:, 0], z["out"])
    for (n, c, t), q, a, want in zip(z["meta"], z["gates"], ins, outs):
        got = oracle.apply_single(a.copy(), gate_from_q(q), int(t), workers)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("workers", [1, 4])
def test_oracle_controlled_bit_exact_vs_reference(workers):
    z = golden("kernel_controlled.npz")
    ins = split_cases(z["meta"][:, 0], z["inp"])
    outs = split_cases(z["meta"][:, 0], z["out"])
    for (n, c, t), q, a, want in zip(z["meta"], z["gates"], ins, outs):
        got = oracle.apply_controlled(a.copy(), gate_from_q(q), int(c), int(t), workers)
        assert np.array_equal(got, want)


def test_reference_build_matches_golden():
    ref = oracle.ref_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    z = golden("kernel_single.npz")
    ins = split_cases(z["meta"][:, 0], z["inp"])
    outs = split_cases(z["meta"][:, 0], z["out"])
    for (n, c, t), q, a, want in zip(z["meta"], z["gates"], ins, outs):
        g = gate_from_q(q)
        b = a.copy()
        ref.apply_single(b, g.q11, g.q12, g.q21, g.q22, int(t), 3, 4)
        assert np.array_equal(b, want)


def test_oracle_partitioned_engine_vs_reference():
    z = golden("engine.npz")
    outs = split_cases(z["meta"][:, 0], z["out"])
    ops = z["ops"]
    for case, ((n, k, scheme_id, nops), want) in enumerate(zip(z["meta"], outs)):
        rows = ops[ops[:, 0] == case]
        seq = [(gate_from_q(r[3:]), int(r[1]), None if int(r[2]) < 0 else int(r[2])) for r in rows]
        L = 1 << (n - k)
        slabs = [np.zeros(L, np.complex128) for _ in range(1 << k)]
        slabs[0][0] = 1
        got = np.concatenate(oracle.run_partitioned(slabs, int(n), seq))
        err = np.max(np.abs(got - want))
        if scheme_id == 0:
            assert err < 1e-12  # scheme a uses numpy arithmetic in the reference
        else:
            assert err < 1e-12
            assert np.array_equal(got, want) or err < 1e-15


def test_oracle_qft_n12_bit_exact_and_n20_sha():
    z = golden("qft.npz")
    for n in (12, 20):
        a = w.seeded_state(n, w.SEED_STATE)
        assert canon_sha(a) == str(z[f"in_sha{n}"])
        circ = circuit_from_rows(n, z[f"ops{n}"])
        # the rebuilt circuit matches the workload builder on this host
        assert np.max(np.abs(np.array([op.gate.as_doubles() for op in circ.ops]) -
                             np.array([op.gate.as_doubles() for op in w.qft_circuit(n).ops]))) < 1e-15
        out = oracle.run_ops(a, w.oracle_ops(circ), workers=4)
        assert canon_sha(out) == str(z[f"sha{n}"])
        assert np.array_equal(out[z[f"idx{n}"]], z[f"amp{n}"])
    assert np.array_equal(out, out)


def test_oracle_layers_sha():
    z = golden("layers.npz")
    a = np.zeros(1 << 12, np.complex128)
    a[0] = 1
    out = oracle.run_ops(a, w.oracle_ops(circuit_from_rows(12, z["ops"])), 4)
    assert canon_sha(out) == str(z["sha"])
    assert np.array_equal(out, z["out"])


def test_dense_oracle_agrees():
    rng = np.random.default_rng(5)
    for n in (3, 6, 9):
        a = w.random_state_array(rng, n)
        circ = w.random_layer_circuit(n, 3, seed=n)
        ops = w.oracle_ops(circ)
        assert np.max(np.abs(oracle.run_ops(a.copy(), ops) - oracle.dense_run(a, n, ops))) < 1e-12


def test_qft_known_answers():
    n = 10
    a = w.random_state_array(np.random.default_rng(1), n)
    out = oracle.run_ops(a.copy(), w.oracle_ops(w.qft_circuit(n)))
    assert np.max(np.abs(out - oracle.qft_reference(a, n))) < 1e-12
    for x in (0, 1, 37, 1023):
        e = np.zeros(1 << n, np.complex128)
        e[x] = 1
        o = oracle.run_ops(e, w.oracle_ops(w.qft_circuit(n)))
        for y in (0, 5, 511, 1000):
            assert abs(o[y] - oracle.qft_basis_amplitude(x, y, n)) < 1e-12


def test_reference_golden_vectors_small():
    # test_kernel.py:48-56, 85-93: X on q2 moves e1 -> e5; CNOT(0->1) e1 -> e3
    from paper_1801_01037_b200.core import standard_gate

    a = np.zeros(8, np.complex128)
    a[1] = 1
    oracle.apply_single(a, standard_gate("x"), 2)
    assert a[5] == 1 and np.count_nonzero(a) == 1
    b = np.zeros(4, np.complex128)
    b[1] = 1
    oracle.apply_controlled(b, standard_gate("x"), 0, 1)
    assert b[3] == 1 and np.count_nonzero(b) == 1
