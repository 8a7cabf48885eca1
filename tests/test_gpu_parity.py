"""GPU parity: libsvb.so kernels vs the CPU oracle and the reference's golden
outputs.  Bar: bit-identical (np.array_equal, zero signs aside) for single
gate kernels and unfused op lists; max-abs <= 1e-12 (the north-star
tolerance) wherever gates are fused or reordered."""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import circuit_from_rows, gate_from_q, golden, split_cases
from paper_1801_01037_b200 import (
    SCHEME_A,
    SCHEME_B,
    Circuit,
    Gate2x2,
    GateOp,
    PartitionPlan,
    StateVector,
    apply_controlled,
    apply_single,
    chunked,
    phase,
    rx,
    ry,
    rz,
    standard_gate,
)
from paper_1801_01037_b200 import _lib, device, engine, workloads as w

pytestmark = pytest.mark.gpu
TOL = 1e-12


def canon_sha(a):
    v = np.ascontiguousarray(a, dtype=np.complex128).view(np.float64) + 0.0
    return hashlib.sha256(v.tobytes()).hexdigest()


def all_gates(rng):
    return [standard_gate(x) for x in "IXYZHST"] + [
        rx(1.1), ry(-0.7), rz(2.5), phase(0.3), w.random_unitary2(rng)]


def test_golden_kernel_single_bit_exact(cuda_ok):
    z = golden("kernel_single.npz")
    ins = split_cases(z["meta"][:, 0], z["inp"])
    outs = split_cases(z["meta"][:, 0], z["out"])
    for (n, c, t), q, a, want in zip(z["meta"], z["gates"], ins, outs):
        s = StateVector(int(n), a.copy())
        apply_single(s, gate_from_q(q), int(t))  # host array -> backend -> C ABI
        assert np.array_equal(s.amps, want)


def test_golden_kernel_controlled_bit_exact(cuda_ok):
    z = golden("kernel_controlled.npz")
    ins = split_cases(z["meta"][:, 0], z["inp"])
    outs = split_cases(z["meta"][:, 0], z["out"])
    for (n, c, t), q, a, want in zip(z["meta"], z["gates"], ins, outs):
        s = StateVector(int(n), a.copy())
        apply_controlled(s, gate_from_q(q), int(c), int(t))
        assert np.array_equal(s.amps, want)


@pytest.mark.parametrize("n", [1, 2, 5, 6, 7, 11, 16])
def test_every_target_every_gate_kind_bit_exact(cuda_ok, n):
    rng = np.random.default_rng(100 + n)
    a = w.random_state_array(rng, n)
    for g in all_gates(rng):
        for t in range(n):
            want = oracle.apply_single(a.copy(), g, t)
            st = device.DeviceState.from_host(a)
            device.apply_single(st, g, t)
            assert np.array_equal(st.to_host().amps, want), (n, t, g)


@pytest.mark.parametrize("n", [2, 6, 7, 12])
def test_every_control_target_pair_bit_exact(cuda_ok, n):
    rng = np.random.default_rng(200 + n)
    a = w.random_state_array(rng, n)
    gates = all_gates(rng)
    for c in range(n):
        for t in range(n):
            if c == t:
                continue
            g = gates[(c * n + t) % len(gates)]
            want = oracle.apply_controlled(a.copy(), g, c, t)
            st = device.DeviceState.from_host(a)
            device.apply_controlled(st, g, c, t)
            assert np.array_equal(st.to_host().amps, want), (n, c, t)


def test_qft20_matches_reference_sha(cuda_ok):
    # config 1: QFT n=20, seeded Gaussian state; reference output hash
    z = golden("qft.npz")
    a = w.seeded_state(20, w.SEED_STATE)
    assert canon_sha(a) == str(z["in_sha20"])
    circ = circuit_from_rows(20, z["ops20"])
    out = device.simulate(circ, a.copy(), fuse=False)
    assert canon_sha(out) == str(z["sha20"])
    assert np.array_equal(out[z["idx20"]], z["amp20"])
    fused = device.simulate(circ, a.copy(), fuse=True)
    assert np.max(np.abs(fused - out)) <= TOL
    st = device.DeviceState.from_host(fused)
    p = device.probs(st).cpu().numpy()
    assert np.max(np.abs(p[z["idx20"]] - z["prob20"])) <= TOL
    assert abs(device.norm2(st) - float(z["norm20"])) <= 1e-12


def test_layers_matches_reference(cuda_ok):
    z = golden("layers.npz")
    circ = circuit_from_rows(12, z["ops"])
    out = device.simulate(circ, None, fuse=False)
    assert canon_sha(out) == str(z["sha"])
    for strict in (True, False):
        f = device.simulate(circ, None, fuse=True, strict_order=strict)
        assert np.max(np.abs(f - z["out"])) <= TOL
        if strict:
            assert np.array_equal(f, z["out"])


@pytest.mark.parametrize("n", [14, 18, 22])
def test_fused_random_layers_vs_oracle(cuda_ok, n):
    circ = w.random_layer_circuit(n, 6, seed=n)
    a = w.random_state_array(np.random.default_rng(n), n)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=8)
    for fuse, strict in ((False, False), (True, True), (True, False)):
        got = device.simulate(circ, a.copy(), fuse=fuse, strict_order=strict)
        err = np.max(np.abs(got - want))
        assert err <= TOL, (fuse, strict, err)
        if not fuse or strict:
            assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [14, 20])
def test_fused_fma_within_tolerance(cuda_ok, n):
    # SVB_RUN_FMA (the bench's default): multiply-adds contracted in fused
    # passes -- not bit-identical, within the north-star 1e-12
    rng = np.random.default_rng(400 + n)
    for circ in (w.random_layer_circuit(n, 8, seed=n), w.qft_circuit(n)):
        a = w.random_state_array(rng, n)
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=8)
        got = device.simulate(circ, a.copy(), fma=True)
        assert np.max(np.abs(got - want)) <= TOL
        st = device.DeviceState.from_host(a)
        device.run_ops(st, circ, fma=True)
        assert np.max(np.abs(st.to_host().amps - want)) <= TOL


@pytest.mark.parametrize("geom", [None, ("12", "5")])
def test_bench_path_deep_circuit_vs_oracle(cuda_ok, geom, monkeypatch):
    # the bench's default path (fused + FMA + JIT: in-register perms, unit
    # folding, scalar extraction with the global factor applied at the end)
    # on the full configs[1] depth -- 200 layers, 7800 ops -- at n = 20, where
    # the oracle finishes in seconds; also the same circuit in two halves
    # (each run_ops applies its own factor).  geom (12, 5): the bench's own
    # geometry at n = 26 (12-qubit tiles, 5 slot bits; n = 20 alone would get
    # 11-qubit tiles); test_gpu_large.py runs n = 26 itself
    if geom is not None:
        monkeypatch.setenv("SVB_JIT_FM", geom[0])
        monkeypatch.setenv("SVB_JIT_FS", geom[1])
    n = 20
    circ = w.random_layer_circuit(n, 200)
    rng = np.random.default_rng(77)
    a = w.random_state_array(rng, n)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=16)
    got = device.simulate(circ, a.copy(), fma=True, jit=True)
    err = np.max(np.abs(got - want))
    assert err <= TOL, err
    st = device.DeviceState.from_host(a)
    half = len(circ.ops) // 2
    device.run_ops(st, circ.ops[:half], fma=True, jit=True)
    device.run_ops(st, circ.ops[half:], fma=True, jit=True)
    assert np.max(np.abs(st.to_host().amps - want)) <= TOL
    assert abs(device.norm2(st) - 1.0) < 1e-12


@pytest.mark.parametrize("fm,fs", [(11, 4), (11, 5), (12, 4), (12, 5), (13, 4), (13, 5)])
def test_jit_tile_sizes_vs_oracle(cuda_ok, fm, fs, monkeypatch):
    # runtime-specialised passes may use 2^12 / 2^13-amplitude tiles (64 /
    # 128 KiB of shared memory) and 16 or 32 amplitudes per thread: every
    # geometry agrees with the oracle, strict order bit-identical to the
    # interpreter's
    monkeypatch.setenv("SVB_JIT_FM", str(fm))
    monkeypatch.setenv("SVB_JIT_FS", str(fs))
    n = 22
    rng = np.random.default_rng(900 + fm)
    circ = w.random_layer_circuit(n, 12, seed=fm)
    a = w.random_state_array(rng, n)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=16)
    got = device.simulate(circ, a.copy(), fma=True, jit=True)
    assert np.max(np.abs(got - want)) <= TOL
    assert device.plan_passes(n, circ, jit=True) <= device.plan_passes(n, circ)
    got = device.simulate(circ, a.copy(), strict_order=True, jit=True)
    assert np.array_equal(got, device.simulate(circ, a.copy(), strict_order=True))


@pytest.mark.parametrize("n", [14, 19])
def test_jit_passes_bit_identical_to_interpreter(cuda_ok, n, monkeypatch):
    # SVB_RUN_JIT compiles each fused pass to straight-line code; on the same
    # plan it must give exactly the interpreter's bits (exact and FMA
    # arithmetic, perms, controls).  JIT plans run X / CNOT in registers by
    # default; SVB_FUSE_REGPERM=1 gives the interpreter that same plan,
    # SVB_JIT_FS=4 its 16 amplitudes per thread (register groups decide which
    # commuting gates meet first), and SVB_JIT_FACTOR=0 turns off the
    # (rounding-level) scalar extraction.
    monkeypatch.setenv("SVB_FUSE_REGPERM", "1")
    monkeypatch.setenv("SVB_JIT_FACTOR", "0")
    monkeypatch.setenv("SVB_JIT_FS", "4")
    monkeypatch.setenv("SVB_FUSE_OUTSIDE", "0")  # tile-uniform predicates: JIT-only plans
    rng = np.random.default_rng(600 + n)
    x = standard_gate("x")
    pool = all_gates(rng) + [x, x, Gate2x2(1, 0, 0, -1j)]
    ops = []
    for _ in range(250):
        g = pool[int(rng.integers(len(pool)))]
        if rng.random() < 0.4:
            c, t = rng.choice(n, size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
        else:
            ops.append(GateOp("single", g, int(rng.integers(n))))
    circs = [Circuit(n, tuple(ops)), w.random_layer_circuit(n, 6, seed=n), w.qft_circuit(n)]
    for circ in circs:
        a = w.random_state_array(rng, n)
        for fma in (False, True):
            ref = device.simulate(circ, a.copy(), fma=fma)
            got = device.simulate(circ, a.copy(), fma=fma, jit=True)
            assert np.array_equal(got, ref), (fma, np.max(np.abs(got - ref)))
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ))
        assert np.max(np.abs(got - want)) <= TOL
        # default plans (JIT: in-register perms; interpreter: deferred) agree
        # to rounding, and strict order stays bit-exact through the JIT
        monkeypatch.delenv("SVB_FUSE_REGPERM")
        monkeypatch.delenv("SVB_JIT_FACTOR")
        monkeypatch.delenv("SVB_JIT_FS")
        got = device.simulate(circ, a.copy(), fma=True, jit=True)
        assert np.max(np.abs(got - want)) <= TOL
        got = device.simulate(circ, a.copy(), strict_order=True, jit=True)
        ref = device.simulate(circ, a.copy(), strict_order=True)
        assert np.array_equal(got, ref)
        monkeypatch.setenv("SVB_FUSE_REGPERM", "1")
        monkeypatch.setenv("SVB_JIT_FACTOR", "0")
        monkeypatch.setenv("SVB_JIT_FS", "4")


@pytest.mark.parametrize("n", [15, 16, 19])
def test_jit_outside_tile_ops_vs_oracle(cuda_ok, n, monkeypatch):
    # specialised passes let Z-type qubits (controls, diagonal targets) stay
    # outside the tile: tile-uniform predicates / per-tile factors, pending
    # swaps whose parity mixes thread and tile bits.  Controlled and diagonal
    # heavy circuits in exact and FMA arithmetic, against the oracle; the plan
    # with them has fewer passes
    rng = np.random.default_rng(700 + n)
    x = standard_gate("x")
    pool = all_gates(rng) + [x, x, x, Gate2x2(1, 0, 0, -1j), rz(0.4), phase(1.3)]
    ops = []
    for _ in range(500):
        g = pool[int(rng.integers(len(pool)))]
        if rng.random() < 0.6:
            c, t = rng.choice(n, size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
        else:
            ops.append(GateOp("single", g, int(rng.integers(n))))
    circs = [Circuit(n, tuple(ops)), w.qft_circuit(n), w.random_layer_circuit(n, 20, seed=n)]
    for circ in circs:
        a = w.random_state_array(rng, n)
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=16)
        for fma in (False, True):
            got = device.simulate(circ, a.copy(), fma=fma, jit=True)
            assert np.max(np.abs(got - want)) <= TOL, (fma, np.max(np.abs(got - want)))
        monkeypatch.setenv("SVB_FUSE_OUTSIDE", "0")
        inside = device.plan_passes(n, circ, jit=True)
        monkeypatch.delenv("SVB_FUSE_OUTSIDE")
        outside = device.plan_passes(n, circ, jit=True)
        assert outside <= inside or circ is circs[0], (outside, inside)


@pytest.mark.parametrize("n", [14, 17])
def test_fused_every_gate_class_strict_bit_exact(cuda_ok, n):
    # every fused opcode family: general / real / anti / Rx / unit-anti gates on
    # any slot, controls on slots and on thread bits, diagonal gates with slot or
    # thread targets, unit (Z, S, S-dagger) and general phases
    rng = np.random.default_rng(300 + n)
    pool = all_gates(rng) + [Gate2x2(1, 0, 0, -1j), Gate2x2(0, 1j, 1j, 0), Gate2x2(0, -1, 1, 0),
                             Gate2x2(1j, 0, 0, 1), rz(0.4)]
    ops = []
    for _ in range(400):
        g = pool[int(rng.integers(len(pool)))]
        if rng.random() < 0.4:
            c, t = rng.choice(n, size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
        else:
            ops.append(GateOp("single", g, int(rng.integers(n))))
    circ = Circuit(n, tuple(ops))
    a = w.random_state_array(rng, n)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ))
    strict = device.simulate(circ, a.copy(), fuse=True, strict_order=True)
    assert np.array_equal(strict, want)
    loose = device.simulate(circ, a.copy(), fuse=True)
    assert np.max(np.abs(loose - want)) <= TOL
    assert device.plan_passes(n, circ, fuse=True) < len(ops)


@pytest.mark.parametrize("n", [14, 15, 19])
def test_fused_permutation_heavy(cuda_ok, n):
    # X / CNOT fold into register-group store maps (incl. direct-to-HBM last
    # groups): mix them densely with arithmetic gates on every qubit
    rng = np.random.default_rng(500 + n)
    x = standard_gate("x")
    pool = [x, x, standard_gate("h"), standard_gate("t"), w.random_unitary2(rng), standard_gate("y")]
    for trial in range(4):
        ops = []
        for _ in range(300):
            g = pool[int(rng.integers(len(pool)))]
            if rng.random() < 0.5:
                c, t = rng.choice(n, size=2, replace=False)
                ops.append(GateOp("controlled", g, int(t), int(c)))
            else:
                ops.append(GateOp("single", g, int(rng.integers(n))))
        circ = Circuit(n, tuple(ops))
        a = w.random_state_array(rng, n)
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ))
        assert np.array_equal(device.simulate(circ, a.copy(), fuse=True, strict_order=True), want), trial
        assert np.max(np.abs(device.simulate(circ, a.copy(), fuse=True) - want)) <= TOL, trial


def test_random_reference_circuits_vs_oracle(cuda_ok):
    # conftest.random_circuit shape (p_controlled = 0.35, Haar gates), n up to 20
    rng = np.random.default_rng(77)
    for _ in range(20):
        n = int(rng.integers(2, 21))
        ops = []
        for _ in range(30):
            g = w.random_unitary2(rng)
            if rng.random() < 0.35:
                c, t = rng.choice(n, size=2, replace=False)
                ops.append(GateOp("controlled", g, int(t), int(c)))
            else:
                ops.append(GateOp("single", g, int(rng.integers(n))))
        circ = Circuit(n, tuple(ops))
        a = w.random_state_array(rng, n)
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ))
        assert np.array_equal(device.simulate(circ, a.copy(), fuse=False), want)
        assert np.max(np.abs(device.simulate(circ, a.copy(), fuse=True) - want)) <= TOL


def test_norm_and_probs(cuda_ok):
    for n in (1, 5, 13, 21):
        a = w.random_state_array(np.random.default_rng(n), n)
        st = device.DeviceState.from_host(a)
        assert abs(device.norm2(st) - float(np.vdot(a, a).real)) <= 1e-12
        p = device.probs(st).cpu().numpy()
        assert np.max(np.abs(p - np.abs(a) ** 2)) <= 1e-15
        assert np.array_equal(p, oracle.probs(a))


def test_edge_cases(cuda_ok):
    # zero state never fires a control (test_kernel.py:96-99); identity; X twice
    st = device.DeviceState.zeros(5)
    device.apply_controlled(st, standard_gate("x"), 4, 2)
    h = st.to_host().amps
    assert h[0] == 1 and np.count_nonzero(h) == 1
    a = w.random_state_array(np.random.default_rng(9), 10)
    st = device.DeviceState.from_host(a)
    for t in range(10):
        device.apply_single(st, standard_gate("i"), t)
    assert np.array_equal(st.to_host().amps, a)
    for _ in range(2):
        device.apply_single(st, standard_gate("x"), 7)
    assert np.array_equal(st.to_host().amps, a)
    # empty op list is a no-op
    device.run_ops(st, [])
    assert np.array_equal(st.to_host().amps, a)
    # invalid arguments raise, never launch
    from paper_1801_01037_b200 import ValidationError

    with pytest.raises(ValidationError):
        device.apply_single(st, standard_gate("x"), 10)
    with pytest.raises(ValidationError):
        device.apply_controlled(st, standard_gate("x"), 3, 3)


def test_launch_counter_moves(cuda_ok):
    before = _lib.launch_count()
    st = device.DeviceState.zeros(12)
    device.apply_single(st, standard_gate("h"), 3)
    import torch

    torch.cuda.synchronize()
    assert _lib.launch_count() == before + 1


# ---- partitioned engine ---------------------------------------------------


def test_engine_vs_reference_golden(cuda_ok):
    z = golden("engine.npz")
    outs = split_cases(z["meta"][:, 0], z["out"])
    ops = z["ops"]
    pos = 0
    for case, ((n, k, scheme_id, nops), want) in enumerate(zip(z["meta"], outs)):
        rows = ops[ops[:, 0] == case]
        circ = Circuit(int(n), tuple(
            GateOp("single" if r[2] < 0 else "controlled", gate_from_q(r[3:]), int(r[1]),
                   None if r[2] < 0 else int(r[2])) for r in rows))
        scheme = (SCHEME_A, SCHEME_B, chunked(2))[int(scheme_id)]
        ds, stats = engine.run_circuit(circ, PartitionPlan(int(n), int(k)), scheme)
        got = engine.gather(ds).amps
        ds.close()
        assert np.max(np.abs(got - want)) <= TOL, case
        if scheme_id == 1:  # scheme b: Python complex arithmetic == C kernel
            assert np.array_equal(got, want), case
        assert [s.messages_sent_per_rank for s in stats] == list(z["msgs"][pos:pos + nops])
        assert [s.bytes_sent_per_rank for s in stats] == list(z["bytes"][pos:pos + nops])
        pos += nops


@pytest.mark.parametrize("fused", [True, "fast"])
def test_engine_fused_seam_vs_reference_golden(cuda_ok, fused):
    """run_circuit(fused=...) (local ops between exchanges as one fused
    svb_run_ops per rank) against the reference's engine goldens: same
    amplitudes (bit-identical for the strict fused mode where the op-by-op
    path is), same per-gate messages and bytes."""
    z = golden("engine.npz")
    outs = split_cases(z["meta"][:, 0], z["out"])
    ops = z["ops"]
    pos = 0
    for case, ((n, k, scheme_id, nops), want) in enumerate(zip(z["meta"], outs)):
        rows = ops[ops[:, 0] == case]
        circ = Circuit(int(n), tuple(
            GateOp("single" if r[2] < 0 else "controlled", gate_from_q(r[3:]), int(r[1]),
                   None if r[2] < 0 else int(r[2])) for r in rows))
        scheme = (SCHEME_A, SCHEME_B, chunked(2))[int(scheme_id)]
        ds, stats = engine.run_circuit(circ, PartitionPlan(int(n), int(k)), scheme, fused=fused)
        got = engine.gather(ds).amps
        ds.close()
        assert np.max(np.abs(got - want)) <= TOL, case
        if scheme_id == 1 and fused is True:
            assert np.array_equal(got, want), case
        assert len(stats) == nops
        assert [s.messages_sent_per_rank for s in stats] == list(z["msgs"][pos:pos + nops])
        assert [s.bytes_sent_per_rank for s in stats] == list(z["bytes"][pos:pos + nops])
        assert all(s.wall_time >= 0 for s in stats)
        pos += nops


def test_engine_fused_seam_large_matches_op_by_op(cuda_ok):
    """A configs[1]-style circuit at n=20 over 4 ranks with a global control
    and target mix: fused (strict) equals op-by-op bit for bit, and the
    rank-bit-controlled local ops (regime iii) are kept per rank."""
    n = 20
    circ = w.random_layer_circuit(n, 6, seed=77)
    a = w.random_state_array(np.random.default_rng(77), n)
    ds0, st0 = engine.run_circuit(circ, PartitionPlan(n, 2), SCHEME_B, initial=a)
    ds1, st1 = engine.run_circuit(circ, PartitionPlan(n, 2), SCHEME_B, initial=a, fused=True)
    g0, g1 = engine.gather(ds0).amps, engine.gather(ds1).amps
    ds0.close()
    ds1.close()
    assert np.array_equal(g0, g1)
    assert [(s.comm_required, s.messages_sent_per_rank, s.bytes_sent_per_rank) for s in st0] == \
        [(s.comm_required, s.messages_sent_per_rank, s.bytes_sent_per_rank) for s in st1]


@pytest.mark.parametrize("k", [1, 2, 3])
def test_engine_partitioned_equals_single_rank(cuda_ok, k):
    n = 16
    circ = w.random_layer_circuit(n, 3, seed=40 + k)
    a = w.random_state_array(np.random.default_rng(k), n)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=8)
    ds, stats = engine.run_circuit(circ, PartitionPlan(n, k), SCHEME_B, initial=a)
    got = engine.gather(ds).amps
    assert np.array_equal(got, want)
    assert any(s.comm_required for s in stats)
    pb = ds.peer_bytes()
    assert all(b > 0 for b in pb)
    ds.close()


def test_engine_known_answers(cuda_ok):
    # test_engine.py:87-95: X on the top qubit at n=3, k=2 swaps the halves
    ds = engine.dist_init(PartitionPlan(3, 2), scheme=SCHEME_B,
                          initial=np.arange(8, dtype=np.complex128))
    engine.dist_apply_scheme_b(ds, standard_gate("x"), 2)
    assert np.array_equal(engine.gather(ds).amps, np.array([4, 5, 6, 7, 0, 1, 2, 3], np.complex128))
    ds.close()
    # test_engine.py:98-109 scheme a pairing
    ds = engine.dist_init(PartitionPlan(4, 2), scheme=SCHEME_A, initial=np.arange(16, dtype=np.complex128))
    engine.dist_apply_scheme_a(ds, standard_gate("x"), 3)
    want = np.array([8, 9, 10, 11, 12, 13, 14, 15, 0, 1, 2, 3, 4, 5, 6, 7], np.complex128)
    assert np.array_equal(engine.gather(ds).amps, want)
    ds.close()


def test_qft_known_answer_partitioned(cuda_ok):
    n, k = 14, 3
    x = 12345
    e = np.zeros(1 << n, np.complex128)
    e[x] = 1
    ds, _ = engine.run_circuit(w.qft_circuit(n), PartitionPlan(n, k), SCHEME_B, initial=e)
    out = engine.gather(ds).amps
    ds.close()
    for y in (0, 1, 77, 4096, 16383):
        assert abs(out[y] - oracle.qft_basis_amplitude(x, y, n)) <= TOL
    assert abs(np.vdot(out, out).real - 1) <= 1e-12


def test_simulate_batch_equals_serial(cuda_ok):
    # svb_host_run_ops_batch (pipelined H2D / run / D2H over three device
    # buffers) returns exactly what one svb_host_run_ops call per state does
    import torch

    n = 20
    circ = w.random_layer_circuit(n, 12, seed=9)
    rng = np.random.default_rng(90)
    states = [w.random_state_array(rng, n) for _ in range(5)]
    serial = [device.simulate(circ, s.copy(), fma=True, jit=True) for s in states]
    pins = [torch.from_numpy(s.copy()).pin_memory().numpy() for s in states]
    outs = [torch.empty(1 << n, dtype=torch.complex128).pin_memory().numpy() for _ in states]
    device.simulate_batch(circ, pins, outs, fma=True, jit=True)
    for got, want in zip(outs, serial):
        assert np.array_equal(got, want)
    inplace = [s.copy() for s in states[:2]]  # pageable, in place, batch smaller than the buffer ring
    device.simulate_batch(circ, inplace, fma=True, jit=True)
    for got, want in zip(inplace, serial):
        assert np.array_equal(got, want)
    assert device.simulate_batch(circ, [], fma=True, jit=True) == []
    device.release_staging()  # buffers come back on the next call
    again = device.simulate_batch(circ, [states[0].copy()], fma=True, jit=True)[0]
    assert np.array_equal(again, serial[0])
    device.release_staging()
    assert np.array_equal(device.simulate(circ, states[1].copy(), fma=True, jit=True), serial[1])


def test_plan_cache_eviction_unloads_and_rebuilds(cuda_ok, monkeypatch):
    # plans beyond the cache bound are dropped with their JIT modules; a
    # circuit seen again is re-planned and recompiled, same results
    monkeypatch.setenv("SVB_PLAN_CACHE_MB", "0")  # keep only the 4 most recent plans
    n = 16
    rng = np.random.default_rng(99)
    a = w.random_state_array(rng, n)
    circs = [w.random_layer_circuit(n, 3, seed=1000 + i) for i in range(7)]
    first = device.simulate(circs[0], a.copy(), fma=True, jit=True)
    for c in circs[1:]:
        device.simulate(c, a.copy(), fma=True, jit=True)
    again = device.simulate(circs[0], a.copy(), fma=True, jit=True)
    assert np.array_equal(again, first)
    want = oracle.run_ops(a.copy(), w.oracle_ops(circs[0]))
    assert np.max(np.abs(again - want)) <= TOL


def test_jit_fast_fuzz_vs_oracle(cuda_ok):
    # the bench's path (JIT, FMA, factor extraction, outside-tile plans,
    # per-thread / per-slot phases, pending swaps) on random circuits drawn
    # from mixed gate pools -- a net for code-generation and compiler
    # regressions
    rng = np.random.default_rng(2024)
    x = standard_gate("x")
    base = [standard_gate(g) for g in "XYZHST"] + [x, x]
    for trial in range(12):
        n = int(rng.integers(15, 21))
        pool = base + [rx(float(rng.uniform(0, 6.3))), ry(float(rng.uniform(0, 6.3))),
                       rz(float(rng.uniform(0, 6.3))), phase(float(rng.uniform(0, 6.3))), w.random_unitary2(rng)]
        p_ctl = float(rng.uniform(0.1, 0.7))
        ops = []
        for _ in range(int(rng.integers(100, 600))):
            g = pool[int(rng.integers(len(pool)))]
            if rng.random() < p_ctl:
                c, t = rng.choice(n, size=2, replace=False)
                ops.append(GateOp("controlled", g, int(t), int(c)))
            else:
                ops.append(GateOp("single", g, int(rng.integers(n))))
        circ = Circuit(n, tuple(ops))
        a = w.random_state_array(rng, n)
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=16)
        got = device.simulate(circ, a.copy(), fma=True, jit=True)
        assert np.max(np.abs(got - want)) <= TOL, (trial, n, np.max(np.abs(got - want)))


@pytest.mark.parametrize("n", [14, 18, 22])
def test_jit_cnot_chains_carry_pending_swaps(cuda_ok, n):
    # CNOT chains a->b->c->... between arithmetic gates: a CNOT from a
    # thread bit onto a slot becomes a pending swap X_k^p; a following CNOT
    # controlled by that slot carries it (X_k CNOT_{k->s} X_k = CNOT_{k->s}
    # X_s), and H / Ry / T on the slots consume or pass through it.  Bench
    # path (FMA + JIT) against the oracle, several seeds and geometries
    x = standard_gate("x")
    for seed in range(6):
        rng = np.random.default_rng(4000 + 10 * n + seed)
        ops = []
        for _ in range(40):
            chain = rng.permutation(n)[: int(rng.integers(3, 8))]
            for a, b in zip(chain[:-1], chain[1:]):
                ops.append(GateOp("controlled", x, int(b), int(a)))
            for q in rng.choice(n, size=int(rng.integers(1, 5)), replace=False):
                g = (standard_gate("h"), ry(float(rng.uniform(0, 6.3))), standard_gate("t"),
                     rx(float(rng.uniform(0, 6.3))), x)[int(rng.integers(5))]
                ops.append(GateOp("single", g, int(q)))
        circ = Circuit(n, tuple(ops))
        a0 = w.random_state_array(rng, n)
        want = oracle.run_ops(a0.copy(), w.oracle_ops(circ), workers=16)
        got = device.simulate(circ, a0.copy(), fma=True, jit=True)
        assert np.max(np.abs(got - want)) <= TOL, (seed, np.max(np.abs(got - want)))


def test_engine_undersized_buffer_is_capacity_error(cuda_ok):
    # test_engine.py:284-288: a scheme-b state has one-amplitude scratch, so a
    # scheme-a exchange (L/2 amplitudes) is refused before any data moves
    from paper_1801_01037_b200 import CapacityError

    plan = PartitionPlan(5, 1)
    ds = engine.dist_init(plan, scheme=SCHEME_B)
    with pytest.raises(CapacityError):
        engine.dist_apply_scheme_a(ds, standard_gate("h"), 4)
    with pytest.raises(CapacityError):
        engine.dist_apply_controlled(ds, standard_gate("x"), 0, 4, scheme=SCHEME_A)
    engine.dist_apply_scheme_b(ds, standard_gate("h"), 4)  # fits
    ds.close()
    ds = engine.dist_init(plan)  # no scheme: full-slab scratch, every protocol runs
    engine.dist_apply_scheme_a(ds, standard_gate("h"), 4)
    ds.close()


def test_engine_reference_positional_order(cuda_ok):
    # dist_init(plan, transport, scheme, execution, strat, kernel_backend) and
    # run_circuit(circuit, plan, scheme, strat, transport, execution, perm,
    # kernel_backend, norm_tol) as engine.py:157-164, 457-467
    from paper_1801_01037_b200 import InMemoryTransport, SEQUENTIAL, ValidationError

    plan = PartitionPlan(6, 1)
    t = InMemoryTransport(2)
    ds = engine.dist_init(plan, t, SCHEME_B, "cooperative", SEQUENTIAL, None)
    assert ds.transport is t and ds.scheme is SCHEME_B
    engine.dist_apply_scheme_b(ds, standard_gate("x"), 5)
    assert t.messages_sent == [32, 32] and t.bytes_sent == [512, 512]
    ds.close()
    with pytest.raises(ValidationError):
        engine.dist_init(plan, InMemoryTransport(4))
    with pytest.raises(ValidationError):
        engine.dist_init(plan, None, SCHEME_B, "bogus")
    circ = w.random_layer_circuit(6, 2, seed=5)
    t2 = InMemoryTransport(2)
    ds, stats = engine.run_circuit(circ, plan, SCHEME_B, SEQUENTIAL, t2, "cooperative", None, None, 1e-10)
    assert sum(t2.messages_sent) == 2 * sum(s.messages_sent_per_rank for s in stats)
    want = oracle.run_ops(_basis0(6), w.oracle_ops(circ))
    assert np.max(np.abs(engine.gather(ds).amps - want)) <= TOL
    ds.close()


def _basis0(n):
    e = np.zeros(1 << n, np.complex128)
    e[0] = 1
    return e


def _swap_ops(pairs):
    x = standard_gate("X")
    ops = []
    for a, b in pairs:
        ops += [GateOp("controlled", x, b, a), GateOp("controlled", x, a, b), GateOp("controlled", x, b, a)]
    return ops


@pytest.mark.parametrize("case", ["reversal", "partial", "gates_then_swaps", "no_network"])
def test_trailing_swap_network_one_pass(cuda_ok, case):
    # a circuit's trailing SWAP network (CNOT triples; the QFT's qubit
    # reversal) runs as one in-place pass (k_swap_bits): pure data movement,
    # so bit-identical to the oracle applying the CNOTs one by one
    n = 16
    rng = np.random.default_rng(77)
    a = w.random_state_array(rng, n)
    h = standard_gate("H")
    pre = []
    if case == "reversal":
        pairs = [(p, n - 1 - p) for p in range(n // 2)]
    elif case == "partial":  # the low block out whole, one swap inside the rest, qubits 6 and 8 fixed
        pairs = [(0, 15), (1, 12), (2, 11), (3, 14), (4, 9), (5, 7), (10, 13)]
    elif case == "gates_then_swaps":
        pre = [GateOp("single", h, 3), GateOp("controlled", standard_gate("X"), 9, 2), GateOp("single", rz(0.4), 15)]
        pairs = [(p, n - 1 - p) for p in range(n // 2)]
    else:  # a low qubit swapped with another low qubit: not a network for the kernel, the usual plan runs
        pairs = [(0, 1), (2, 13), (3, 12), (4, 11)]
    circ = Circuit(n, tuple(pre + _swap_ops(pairs)))
    arr, nops = _lib.ops_array(circ.ops)
    tail = _lib.load().svb_swap_suffix(n, arr, nops)
    assert tail == (0 if case == "no_network" else 3 * len(pairs))
    want = oracle.run_ops(a.copy(), w.oracle_ops(circ))
    for kw in (dict(fuse=True), dict(fuse=True, fma=True, jit=True)):
        got = device.simulate(circ, a.copy(), **kw)
        if pre:
            assert np.max(np.abs(got - want)) <= TOL
        else:
            assert np.array_equal(got, want)
    # the QFT of a basis state through the same path: exact known answers
    x0 = 4321
    e = np.zeros(1 << n, np.complex128)
    e[x0] = 1
    out = device.simulate(w.qft_circuit(n), e, fma=True, jit=True)
    for y in (0, 1, 77, 4096, 65535):
        assert abs(out[y] - oracle.qft_basis_amplitude(x0, y, n)) <= TOL
