"""Multi-process partitioned engine on CPU: world_size 2 and 4 over gloo.

Exercises paper_1801_01037_b200.dist.DistEngine's orchestration (partner
rule, chunk-pipelined send/recv, control packing, the three controlled
regimes, diagonal elision) with a checker-backed compute object; the result
gathered on rank 0 must equal the op-by-op oracle bit for bit.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _circuit(n, k, seed):
    from paper_1801_01037_b200 import Circuit, GateOp, phase, rz, standard_gate
    from paper_1801_01037_b200 import workloads as w

    rng = np.random.default_rng(seed)
    b = n - k
    ops = []
    for _ in range(40):
        kind = rng.integers(6)
        g = [w.random_unitary2(rng), standard_gate("x"), standard_gate("h"), phase(0.7),
             rz(1.3), standard_gate("s")][int(rng.integers(6))]
        if kind == 0:  # local single
            ops.append(GateOp("single", g, int(rng.integers(b))))
        elif kind == 1:  # global single
            ops.append(GateOp("single", g, int(rng.integers(b, n))))
        elif kind == 2:  # regime ii: local control, global target
            ops.append(GateOp("controlled", g, int(rng.integers(b, n)), int(rng.integers(b))))
        elif kind == 3:  # regime iii: global control, local target
            ops.append(GateOp("controlled", g, int(rng.integers(b)), int(rng.integers(b, n))))
        elif kind == 4 and k > 1:  # global control, global target
            c, t = rng.choice(np.arange(b, n), size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
        else:  # local controlled
            c, t = rng.choice(b, size=2, replace=False)
            ops.append(GateOp("controlled", g, int(t), int(c)))
    return Circuit(n, tuple(ops))


def _worker(rank, world, port, n, chunk, elide, layout, queue):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_compute import CpuCompute
        from paper_1801_01037_b200 import workloads as w
        from paper_1801_01037_b200.dist import DistEngine

        k = world.bit_length() - 1
        a0 = w.seeded_state(n, 5)
        circ = _circuit(n, k, seed=n * 10 + world)
        eng = DistEngine(n, compute=CpuCompute(), initial=a0, chunk=chunk, elide_diagonal=elide, layout=layout)
        eng.run(circ)
        nrm = eng.norm2()
        full = eng.gather()
        if rank == 0:
            import oracle

            want = oracle.run_ops(a0.copy(), w.oracle_ops(circ))
            queue.put((bool(np.array_equal(full, want)), float(np.max(np.abs(full - want))), nrm,
                       eng.stats.exchanges + eng.stats.swaps, eng.stats.elided))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,chunk,elide,layout", [(2, 9, 16, True, False), (2, 9, 1 << 20, False, False),
                                                        (4, 10, 7, True, False), (4, 8, 3, False, False),
                                                        (2, 9, 16, True, True), (4, 10, 7, True, True),
                                                        (4, 8, 3, False, True)])
def test_dist_engine_matches_oracle(world, n, chunk, elide, layout):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, chunk, elide, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    equal, err, nrm, exchanges, elided = q.get(timeout=5)
    assert equal, err
    assert abs(nrm - 1.0) < 1e-12
    assert exchanges > 0
    if not elide:
        assert elided == 0


def _worker_peer_fallback(rank, world, port, n, queue):
    # peer transport requested, but one rank cannot export its slab (e.g. a
    # VMM-backed allocation): every rank must fall back to send/recv together
    # (no rank left waiting in a collective), and the run must still be exact
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_compute import CpuCompute
        from paper_1801_01037_b200 import workloads as w
        from paper_1801_01037_b200.dist import DistEngine

        class NoExport(CpuCompute):
            def ipc_handle(self, slab):
                if rank == world - 1:
                    raise RuntimeError("cudaIpcGetMemHandle: invalid argument")
                return b"handle"

            def ipc_open(self, h):  # never reached: the failure is seen first
                raise AssertionError("ipc_open after a failed export")

        k = world.bit_length() - 1
        a0 = w.seeded_state(n, 6)
        circ = _circuit(n, k, seed=77)
        eng = DistEngine(n, compute=NoExport(), initial=a0, chunk=16, peer=True)
        assert not eng.peer
        eng.run(circ)
        full = eng.gather()
        if rank == 0:
            import oracle

            want = oracle.run_ops(a0.copy(), w.oracle_ops(circ))
            queue.put(bool(np.array_equal(full, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dist_engine_peer_export_failure_falls_back_together(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_peer_fallback, args=(r, world, port, 9, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5)


def _worker_stats(rank, world, port, n, scheme_name, queue):
    # DistEngine.run_with_stats: per-gate GateStats of the multi-process
    # engine equal the reference protocol's accounting (engine.protocol_stats,
    # pinned to the reference's own run_circuit by test_host.py), and the
    # state still matches the oracle
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_compute import CpuCompute
        from paper_1801_01037_b200 import engine, time_ratio, workloads as w
        from paper_1801_01037_b200.dist import DistEngine
        from paper_1801_01037_b200.partition import SCHEME_A, SCHEME_B, PartitionPlan, chunked

        scheme = {"a": SCHEME_A, "b": SCHEME_B, "c4": chunked(4)}[scheme_name]
        k = world.bit_length() - 1
        a0 = w.seeded_state(n, 8)
        circ = _circuit(n, k, seed=n + world)
        eng = DistEngine(n, compute=CpuCompute(), initial=a0, chunk=8)
        stats = eng.run_with_stats(circ, scheme)
        assert eng.run_with_stats(type(circ)(n, ()), scheme) == []  # empty circuit
        eng.run(type(circ)(n, ()))
        full = eng.gather()
        if rank == 0:
            import oracle

            want = oracle.run_ops(a0.copy(), w.oracle_ops(circ))
            ref = engine.protocol_stats(circ, PartitionPlan(n, k), scheme)
            got = [(s.messages_sent_per_rank, s.bytes_sent_per_rank) for s in stats]
            comm = [s for s in stats if s.comm_required]
            local = [s for s in stats if not s.comm_required]
            ratio = time_ratio(comm[0], local[0])
            queue.put((bool(np.array_equal(full, want)), got == ref, len(stats) == len(circ.ops), ratio > 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,scheme", [(2, "b"), (4, "a"), (4, "c4")])
def test_dist_engine_per_gate_stats(world, scheme):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_stats, args=(r, world, port, 9, scheme, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) == (True, True, True, True)


def _worker_layout_runs(rank, world, port, n, queue):
    # the layout engine keeps its global<->local transpositions across runs
    # (restored only when the state is read in logical order): three runs,
    # then one op through apply() (which restores the layout first), then
    # gather -- equal to the oracle applying the same ops in order
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_compute import CpuCompute
        from paper_1801_01037_b200 import GateOp, standard_gate, workloads as w
        from paper_1801_01037_b200.dist import DistEngine

        k = world.bit_length() - 1
        a0 = w.seeded_state(n, 9)
        circ = _circuit(n, k, seed=5 * n + world)
        qft = w.qft_circuit(n)
        eng = DistEngine(n, compute=CpuCompute(), initial=a0, chunk=8, layout=True)
        eng.run(circ)
        eng.run(qft)
        eng.run(circ)
        parked = eng._pi != tuple(range(n))
        extra = GateOp("single", standard_gate("h"), n - 1)
        eng.apply(extra)
        full = eng.gather()
        if rank == 0:
            import oracle

            want = a0.copy()
            for c in (circ, qft, circ):
                want = oracle.run_ops(want, w.oracle_ops(c))
            want = oracle.run_ops(want, [(extra.gate, extra.target, None)])
            queue.put((bool(np.max(np.abs(full - want)) <= 1e-12), parked))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_dist_engine_layout_persists_across_runs(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_layout_runs, args=(r, world, port, 10, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok, parked = q.get(timeout=5)
    assert ok
    assert parked  # the layout really was left permuted between runs
