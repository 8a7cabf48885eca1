"""Dense verifier on the GPU (paper_1801_01037_b200.dense; the reference's
oracle.py API): embeddings bit-identical to the reference's
kron / index-write construction, products within 1e-12 of the oracle,
row partitions bit-identical to the plain product, the reference's errors."""

import numpy as np
import pytest

import oracle
from paper_1801_01037_b200 import CapacityError, Circuit, GateOp, StateVector, ValidationError, dense, device
from paper_1801_01037_b200 import standard_gate, workloads as w

TOL = 1e-12


def ref_embed_single(g, i, n):  # oracle.py:83-96, restated
    lower = np.eye(1 << i, dtype=np.complex128)
    upper = np.eye(1 << (n - 1 - i), dtype=np.complex128)
    return np.kron(upper, np.kron(np.array([[g.q11, g.q12], [g.q21, g.q22]], np.complex128), lower))


def ref_embed_controlled(g, c, t, n):  # oracle.py:98-116, restated
    dim = 1 << n
    e = np.eye(dim, dtype=np.complex128)
    j = np.arange(dim)
    base = j[((j >> t) & 1 == 0) & ((j >> c) & 1 == 1)]
    mate = base | (1 << t)
    e[base, base], e[base, mate], e[mate, base], e[mate, mate] = g.q11, g.q12, g.q21, g.q22
    return e


@pytest.mark.gpu
def test_embeddings_bit_identical(cuda_ok):
    rng = np.random.default_rng(3)
    for n in (1, 3, 7):
        for i in range(n):
            g = w.random_unitary2(rng)
            assert np.array_equal(dense.embed_single(g, i, n).to_host(), ref_embed_single(g, i, n))
    n = 6
    for c in range(n):
        for t in range(n):
            if c != t:
                g = w.random_unitary2(rng)
                assert np.array_equal(dense.embed_controlled(g, c, t, n).to_host(), ref_embed_controlled(g, c, t, n))


@pytest.mark.gpu
def test_matvec_and_partitions(cuda_ok):
    rng = np.random.default_rng(4)
    for n in (4, 9, 12):
        s = StateVector(n, w.random_state_array(rng, n))
        g = w.random_unitary2(rng)
        c, t = 0, n - 1
        u = dense.embed_controlled(g, c, t, n)
        got = dense.matvec(u, s)
        want = oracle.apply_controlled(s.amps.copy(), g, c, t)
        assert np.max(np.abs(got.amps - want)) <= TOL
        for kappa in range(0, n + 1, max(1, n // 3)):
            part, rep = dense.matvec_partitioned(u, s, kappa)
            assert np.array_equal(part.amps, got.amps)
            assert rep.p == 1 << kappa and rep.rows_per_rank == 1 << (n - kappa)


@pytest.mark.gpu
def test_oracle_run_matches_engine_and_oracle(cuda_ok):
    rng = np.random.default_rng(5)
    n = 8
    ops = []
    for _ in range(60):
        g = w.random_unitary2(rng)
        if rng.random() < 0.4:
            c, t = rng.choice(n, size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
        else:
            ops.append(GateOp("single", g, int(rng.integers(n))))
    circ = Circuit(n, tuple(ops))
    got = dense.oracle_run(circ).amps
    zero = np.zeros(1 << n, np.complex128)
    zero[0] = 1.0
    assert np.max(np.abs(got - oracle.run_ops(zero.copy(), w.oracle_ops(circ)))) <= TOL
    assert np.max(np.abs(got - device.simulate(circ, None))) <= TOL
    # reference known answer (test_oracle.py:175-184): H then CNOT -> Bell pair
    bell = dense.oracle_run(Circuit(2, (GateOp("single", standard_gate("h"), 0),
                                        GateOp("controlled", standard_gate("x"), 1, 0)))).amps
    assert np.allclose(bell, [2 ** -0.5, 0, 0, 2 ** -0.5], atol=1e-15)


@pytest.mark.gpu
def test_dense_errors_like_reference(cuda_ok):
    g = standard_gate("x")
    with pytest.raises(CapacityError):
        dense.embed_single(g, 0, 13)
    with pytest.raises(CapacityError):
        dense.embed_single(g, 0, 0)
    with pytest.raises(ValidationError):
        dense.embed_single(g, 3, 3)
    with pytest.raises(ValidationError):
        dense.embed_controlled(g, 1, 1, 3)
    with pytest.raises(ValidationError):
        dense.embed_controlled(g, 3, 0, 3)
    with pytest.raises(ValidationError):
        dense.matvec(dense.embed_single(g, 0, 3), StateVector(2, np.array([1, 0, 0, 0], np.complex128)))


def test_matvec_cost_arithmetic():
    # oracle.py:143-157 on CPU (no device work)
    r = dense.matvec_cost(10, 3)
    assert (r.p, r.rows_per_rank) == (8, 128)
    assert r.per_rank_matrix_bytes == 128 * 1024 * 16
    assert r.replicated_vector_bytes == 8 * 1024 * 16
    with pytest.raises(ValidationError):
        dense.matvec_cost(4, 5)
