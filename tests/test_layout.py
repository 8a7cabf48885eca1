"""Qubit relabeling, against the reference's own known
answers (pkg/tests/test_layout.py) and, on the GPU, the device gather and a
relabeled partitioned run vs the oracle."""

import itertools

import numpy as np
import pytest

import oracle
from paper_1801_01037_b200 import SCHEME_B, Circuit, GateOp, PartitionPlan, StateVector, ValidationError, standard_gate
from paper_1801_01037_b200 import workloads as w
from paper_1801_01037_b200.layout import (
    QubitPermutation,
    gate_histogram,
    identity_perm,
    optimize_layout,
    permute_state,
    permuted_stride,
)

SWAP_12 = QubitPermutation.from_phys((0, 2, 1))


def test_permutation_algebra():
    assert identity_perm(3).phys_to_logical == (0, 1, 2)
    with pytest.raises(ValidationError):
        QubitPermutation.from_phys((0, 0, 1))
    with pytest.raises(ValidationError):
        QubitPermutation((0, 1, 2), (0, 2, 1))
    p = QubitPermutation.from_phys((2, 0, 3, 1))
    q = p.inverse()
    assert tuple(q.phys_to_logical[p.phys_to_logical[i]] for i in range(4)) == (0, 1, 2, 3)
    assert (permuted_stride(SWAP_12, 2), permuted_stride(SWAP_12, 1), permuted_stride(SWAP_12, 0)) == (2, 4, 1)


def test_permute_state_storage_order_golden():
    # test_layout.py:76-80
    s = StateVector(3, np.arange(8, dtype=np.complex128) / np.linalg.norm(np.arange(8)))
    out = permute_state(s, SWAP_12)
    assert np.array_equal(out.amps, s.amps[[0, 1, 4, 5, 2, 3, 6, 7]])
    rng = np.random.default_rng(42)
    for phys in itertools.permutations(range(3)):
        p = QubitPermutation.from_phys(phys)
        s = StateVector(3, w.random_state_array(rng, 3))
        assert np.array_equal(permute_state(permute_state(s, p), p.inverse()).amps, s.amps)


def test_histogram_and_optimize_layout_golden():
    circ = Circuit(3, (GateOp("single", standard_gate("h"), 0), GateOp("controlled", standard_gate("x"), 2, 1),
                       GateOp("single", standard_gate("x"), 2)))
    assert gate_histogram(circ) == [1, 1, 2]
    assert optimize_layout([5, 1, 7], 1).phys_to_logical == (0, 2, 1)
    assert optimize_layout([3, 3, 3, 3], 2).phys_to_logical == (0, 1, 2, 3)
    perm = optimize_layout([4, 0, 9, 0], 2)
    assert sorted(perm.phys_to_logical[2:]) == [1, 3]
    rng = np.random.default_rng(43)
    for n in range(2, 7):
        for k in range(1, n):
            for _ in range(10):
                counts = [int(v) for v in rng.integers(0, 9, size=n)]
                perm = optimize_layout(counts, k)
                got = sum(counts[q] for q in perm.phys_to_logical[n - k:])
                best = min(sum(counts[q] for q in sub) for sub in itertools.combinations(range(n), k))
                assert got == best


def test_layout_changes_protocol_accounting():
    # test_layout.py:165-180 through the host accounting model
    from paper_1801_01037_b200 import engine

    plan = PartitionPlan(3, 1)
    on_q2 = Circuit(3, (GateOp("single", standard_gate("h"), SWAP_12.logical_to_phys[2]),))
    on_q1 = Circuit(3, (GateOp("single", standard_gate("h"), SWAP_12.logical_to_phys[1]),))
    assert engine.protocol_stats(on_q2, plan, SCHEME_B) == [(0, 0)]
    assert engine.protocol_stats(on_q1, plan, SCHEME_B) == [(plan.local_len, 16 * plan.local_len)]


@pytest.mark.gpu
def test_device_permute_matches_host(cuda_ok):
    from paper_1801_01037_b200 import device

    rng = np.random.default_rng(7)
    for n in (3, 9, 17):
        a = w.random_state_array(rng, n)
        p = QubitPermutation.from_phys(tuple(int(v) for v in rng.permutation(n)))
        got = permute_state(device.DeviceState.from_host(a), p).to_host().amps
        assert np.array_equal(got, permute_state(StateVector(n, a), p).amps)


@pytest.mark.gpu
def test_relabeled_partitioned_run_matches_oracle(cuda_ok):
    from paper_1801_01037_b200 import engine

    rng = np.random.default_rng(45)
    for _ in range(12):
        n = int(rng.integers(3, 11))
        k = int(rng.integers(0, min(3, n - 1) + 1))
        circ = w.random_layer_circuit(n, 3, seed=int(rng.integers(1 << 30)))
        perm = optimize_layout(gate_histogram(circ), k) if rng.random() < 0.5 else \
            QubitPermutation.from_phys(tuple(int(v) for v in rng.permutation(n)))
        ds, _ = engine.run_circuit(circ, PartitionPlan(n, k), SCHEME_B, perm=perm)
        logical = permute_state(engine.gather(ds), perm.inverse())
        ds.close()
        a = np.zeros(1 << n, np.complex128)
        a[0] = 1
        want = oracle.run_ops(a, w.oracle_ops(circ))
        assert np.max(np.abs(logical.amps - want)) <= 1e-12
