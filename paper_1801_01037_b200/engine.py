"""Partitioned execution over rank slabs in HBM (mirrors pkg/src/svsim/engine.py).

Same public surface as the reference engine -- ``dist_init``, ``gather``,
``dist_apply_local``, ``dist_apply_scheme_a/b``, ``dist_apply_chunked``,
``dist_apply_controlled``, ``run_circuit``, ``GateStats``, ``time_ratio``
(engine.py:157-521) -- but every rank's slab is a CUDA tensor and every
update is a libsvb.so kernel driven through one ``svb_dist`` handle:

* local gates: one kernel per rank, ranks' streams run concurrently
  (the reference sweeps ranks one after another, engine.py:348-356);
* global-target gates: the fused peer-memory pair kernel -- the lower rank
  of each pair updates pairs j < L/2, the upper rank j >= L/2, each reading
  and writing the partner slab directly (NVLink P2P when the ranks sit on
  different GPUs);
* the three controlled regimes of engine.py:415-450.

All three reference protocols compute the same amplitudes (engine.py:160-184
asserts agreement), so the scheme no longer changes the data path; it keeps
its meaning for the accounting: ``GateStats`` reports the messages/bytes the
reference protocol would send per rank (exact formulas, partition.py here),
and ``peer_bytes`` what the fused kernel actually moved.

Ranks may share a GPU (emulated ranks; every exchange is then a same-device
pair kernel) or be spread over several GPUs of one process.  The
multi-process, one-GPU-per-process engine is ``paper_1801_01037_b200.dist``.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import Circuit, Gate2x2, StateVector
from .errors import CapacityError, ContractViolation, ValidationError
from .partition import (
    SCHEME_A,
    SCHEME_B,
    CommScheme,
    PartitionPlan,
    needs_comm,
    protocol_accounting,
)


@dataclass(frozen=True)
class GateStats:
    """Per-gate accounting (engine.py:143-154): messages/bytes are the max over
    ranks of what the reference protocol sends; wall_time is device-synchronised
    wall time of the gate."""

    qubit: int
    control: int | None
    comm_required: bool
    messages_sent_per_rank: int
    bytes_sent_per_rank: int
    wall_time: float


class PeerTransport:
    """Accounting face of the transport (engine.py:57-120's counters).

    The reference's InMemoryTransport moves every message through Python
    FIFOs; here amplitudes move GPU to GPU through peer memory inside the
    pair kernels, so the object keeps only what callers read from it: the
    rank count and the per-sender message / byte counters of the reference
    protocol (exact formulas, partition.protocol_accounting).  Exported as
    ``InMemoryTransport`` too, so reference code that builds one and passes
    it to dist_init / run_circuit keeps working."""

    def __init__(self, nranks: int, record_log: bool = False):
        if nranks < 1:
            raise ValidationError(f"need at least one rank, got {nranks}")
        self.nranks = int(nranks)
        self.messages_sent = [0] * self.nranks
        self.bytes_sent = [0] * self.nranks
        self.log: list[tuple[int, int, int]] | None = [] if record_log else None

    def count(self, src: int, dst: int, messages: int, nbytes: int) -> None:
        self.messages_sent[src] += messages
        self.bytes_sent[src] += nbytes
        if self.log is not None and messages:
            self.log.append((src, dst, nbytes))


InMemoryTransport = PeerTransport


class DistState:
    """2^k slabs plus the native handle that drives them (engine.py:132-140)."""

    def __init__(self, plan: PartitionPlan, scheme: CommScheme | None, slabs, devices,
                 transport: PeerTransport | None = None, buffer_amps: int | None = None,
                 execution: str = "cooperative", strat=None, kernel_backend: str | None = None):
        self.plan = plan
        self.scheme = scheme
        self.slabs = slabs
        self.devices = list(devices)
        self.transport = transport if transport is not None else PeerTransport(plan.p)
        # per-rank protocol scratch the reference would allocate (engine.py:179):
        # exchanges whose scheme needs more raise CapacityError like the reference
        self.buffer_amps = plan.local_len if buffer_amps is None else buffer_amps
        self.execution = execution
        self.strat = strat
        self.kernel_backend = kernel_backend
        lib = _lib.load()
        p = plan.p
        dev_arr = (ctypes.c_int * p)(*self.devices)
        slab_arr = (ctypes.c_void_p * p)(*[s.data_ptr() for s in slabs])
        h = ctypes.c_void_p()
        import torch

        torch.cuda.synchronize()
        _lib.check(lib.svb_dist_create(plan.n, plan.k, dev_arr, slab_arr, ctypes.byref(h)), "dist_init")
        self._h = h

    @property
    def messages_sent(self) -> list[int]:
        return self.transport.messages_sent

    @property
    def bytes_sent(self) -> list[int]:
        return self.transport.bytes_sent

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise ContractViolation("distributed state already closed")
        return self._h

    def sync(self) -> None:
        _lib.check(_lib.load().svb_dist_sync(self.handle), "sync")

    def peer_bytes(self) -> list[int]:
        arr = (ctypes.c_int64 * self.plan.p)()
        ex = ctypes.c_int64()
        _lib.check(_lib.load().svb_dist_stats(self.handle, ctypes.byref(ex), arr), "stats")
        return list(arr)

    def close(self) -> None:
        if self._h is not None:
            _lib.load().svb_dist_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def dist_init(plan: PartitionPlan, transport: PeerTransport | None = None, scheme: CommScheme | None = None,
              execution: str = "cooperative", strat=None, kernel_backend: str | None = None, *,
              devices=None, initial=None) -> DistState:
    """|0...0> (or `initial`, host array / StateVector) across the plan's ranks
    (engine.py:157-185; same positional order -- plan, transport, scheme,
    execution, strat, kernel_backend).  With a scheme, each rank's protocol
    scratch is that scheme's requirement (exchanges of a scheme needing more
    raise CapacityError); without one, a full slab.  Keyword-only extras:
    devices (CUDA ordinal per rank, default all on the current device) and
    initial."""
    import torch

    _lib.load()
    if execution not in ("cooperative", "threads"):
        raise ValidationError(f"unknown execution mode {execution!r}")
    if transport is None:
        transport = PeerTransport(plan.p)
    elif transport.nranks != plan.p:
        raise ValidationError(f"transport has {transport.nranks} ranks, plan needs {plan.p}")
    if devices is None:
        devices = [torch.cuda.current_device()] * plan.p
    devices = list(devices)
    if len(devices) != plan.p:
        raise ValidationError(f"need {plan.p} device ordinals, got {len(devices)}")
    buf_amps = plan.local_len if scheme is None else max(scheme.buffer_amps(plan), 1)
    L = plan.local_len
    slabs = []
    if initial is not None:
        amps = initial.amps if isinstance(initial, StateVector) else np.ascontiguousarray(initial, np.complex128)
        if amps.shape[0] != (1 << plan.n):
            raise ValidationError(f"initial state must have 2**{plan.n} amplitudes")
        for r in range(plan.p):
            slabs.append(torch.from_numpy(amps[r * L:(r + 1) * L].copy()).to(f"cuda:{devices[r]}"))
    else:
        for r in range(plan.p):
            s = torch.zeros(L, dtype=torch.complex128, device=f"cuda:{devices[r]}")
            if r == 0:
                s[0] = 1.0
            slabs.append(s)
    return DistState(plan, scheme, slabs, devices, transport, buf_amps, execution, strat, kernel_backend)


def gather(ds: DistState) -> StateVector:
    """Concatenate slabs in rank order (engine.py:188-192) on the host."""
    ds.sync()
    return StateVector(ds.plan.n, np.concatenate([s.cpu().numpy() for s in ds.slabs]), validate=False)


def _account(ds: DistState, scheme: CommScheme, t: int, cbit: int | None, participants) -> None:
    plan = ds.plan
    gb = t - (plan.n - plan.k)
    for r in range(plan.p):
        if participants is not None and r not in participants:
            continue
        q = r ^ (1 << gb)
        m, b = protocol_accounting(plan, scheme, r < q, cbit)
        ds.transport.count(r, q, m, b)


def protocol_stats(circuit: Circuit, plan: PartitionPlan, scheme: CommScheme | None) -> list[tuple[int, int]]:
    """Host-only: per-op (messages, bytes) max over ranks that run_circuit's
    GateStats report for this circuit (engine.py:495-505 semantics)."""
    boundary = plan.n - plan.k
    out = []
    for op in circuit.ops:
        t, c = op.target, op.control
        if t < boundary:
            out.append((0, 0))
            continue
        if scheme is None:
            raise ValidationError("communicating target requires a scheme")
        gb = t - boundary
        parts = None
        cbit = None
        if c is not None:
            if c >= boundary:
                parts = {r for r in range(plan.p) if (r >> (c - boundary)) & 1}
            else:
                cbit = c
        best = (0, 0)
        msgs_max = bytes_max = 0
        for r in range(plan.p):
            if parts is not None and r not in parts:
                continue
            m, b = protocol_accounting(plan, scheme, r < (r ^ (1 << gb)), cbit)
            msgs_max, bytes_max = max(msgs_max, m), max(bytes_max, b)
        best = (msgs_max, bytes_max)
        out.append(best)
    return out


def _check_capacity(ds: DistState, scheme: CommScheme) -> None:
    """engine.py:372-377."""
    need = scheme.buffer_amps(ds.plan)
    if need > ds.buffer_amps:
        raise CapacityError(f"rank buffers hold {ds.buffer_amps} amplitudes, scheme needs {need}")


def dist_apply_local(ds: DistState, g: Gate2x2, i: int, strat=None) -> None:
    """engine.py:348-356."""
    if needs_comm(ds.plan, i):
        raise ContractViolation(f"qubit {i} spans ranks for n={ds.plan.n}, k={ds.plan.k}; use a scheme")
    _lib.check(_lib.load().svb_dist_apply_1q(ds.handle, _lib.gate_array(g), int(i)), "dist_apply_local")


def _exchange(ds: DistState, g: Gate2x2, i: int, scheme: CommScheme) -> None:
    plan = ds.plan
    if not needs_comm(plan, i):
        raise ContractViolation(f"qubit {i} is rank-local for n={plan.n}, k={plan.k}; use dist_apply_local")
    _check_capacity(ds, scheme)
    _lib.check(_lib.load().svb_dist_apply_1q(ds.handle, _lib.gate_array(g), int(i)), "exchange")
    _account(ds, scheme, i, None, None)


def dist_apply_scheme_a(ds: DistState, g: Gate2x2, i: int) -> None:
    _exchange(ds, g, i, SCHEME_A)


def dist_apply_scheme_b(ds: DistState, g: Gate2x2, i: int) -> None:
    _exchange(ds, g, i, SCHEME_B)


def dist_apply_chunked(ds: DistState, g: Gate2x2, i: int, m: int) -> None:
    _exchange(ds, g, i, CommScheme("chunked", m))


def dist_apply_controlled(ds: DistState, g: Gate2x2, c: int, t: int,
                          scheme: CommScheme | None = None) -> None:
    """engine.py:415-450: three regimes, dispatched natively."""
    plan = ds.plan
    for name, idx in (("control", c), ("target", t)):
        if not (0 <= idx < plan.n):
            raise ValidationError(f"{name} bit {idx} out of range for n={plan.n}")
    if c == t:
        raise ValidationError("control and target must differ")
    scheme = scheme if scheme is not None else ds.scheme
    boundary = plan.n - plan.k
    if t >= boundary:
        if scheme is None:
            raise ValidationError("communicating target requires a scheme")
        _check_capacity(ds, scheme)
    _lib.check(_lib.load().svb_dist_apply_c1q(ds.handle, _lib.gate_array(g), int(c), int(t)),
               "dist_apply_controlled")
    if t >= boundary:
        if c >= boundary:
            parts = {r for r in range(plan.p) if (r >> (c - boundary)) & 1}
            _account(ds, scheme, t, None, parts)
        else:
            _account(ds, scheme, t, c, None)


def dist_norm2(ds: DistState) -> float:
    out = ctypes.c_double()
    _lib.check(_lib.load().svb_dist_norm2(ds.handle, ctypes.byref(out)), "norm2")
    return out.value


def _run_fused(ds: DistState, circuit: Circuit, l2p, norm_tol: float | None, fast: bool) -> list[GateStats]:
    """run_circuit(fused=...): the local ops between two global-target gates
    run as ONE svb_run_ops per rank (multi-gate HBM passes; each rank gets
    its own list -- a rank-bit control keeps or drops the op per rank,
    regime iii); global-target gates go through the pair kernels as in the
    op-by-op path.  GateStats keep the reference's exact messages / bytes per
    gate; a batch's measured wall time is split evenly over its ops (per-gate
    times inside a fused pass do not exist), exchanges are timed one by one.
    fast=False: strict order, reference arithmetic -- bit-identical to the
    op-by-op path; fast=True: FMA + runtime-specialised passes (<= 1e-12)."""
    import torch

    from .core import GateOp

    lib = _lib.load()
    plan = ds.plan
    boundary = plan.n - plan.k
    flags = _lib.run_flags(fuse=True, fma=True, jit=True) if fast else _lib.run_flags(fuse=True, strict_order=True)
    stats: list[GateStats | None] = [None] * len(circuit.ops)
    pending: list[list] = [[] for _ in range(plan.p)]
    batch: list[int] = []  # op positions in the current local batch

    def flush():
        if not batch:
            return
        ds.sync()
        t0 = time.perf_counter()
        for r in range(plan.p):
            if not pending[r]:
                continue
            slab = ds.slabs[r]
            with torch.cuda.device(slab.device):
                arr, nops = _lib.ops_array(tuple(pending[r]))
                _lib.check(lib.svb_run_ops(ctypes.c_void_p(slab.data_ptr()), slab.shape[0], arr, nops, flags,
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                           "run_circuit(fused)")
        for d in sorted(set(ds.devices)):
            torch.cuda.synchronize(d)
        wall = (time.perf_counter() - t0) / len(batch)
        for pos in batch:
            op = circuit.ops[pos]
            stats[pos] = GateStats(op.target, op.control, False, 0, 0, wall)
        batch.clear()
        for lst in pending:
            lst.clear()
        if norm_tol is not None:
            drift = abs(dist_norm2(ds) - 1.0)
            if drift > norm_tol:
                raise ValidationError(f"norm drifted by {drift:.3e} after gate {pos}")

    for pos, op in enumerate(circuit.ops):
        tbit = l2p[op.target]
        cbit = l2p[op.control] if op.control is not None else None
        if tbit < boundary:
            for r in range(plan.p):
                if cbit is None:
                    pending[r].append(GateOp("single", op.gate, tbit))
                elif cbit >= boundary:  # regime iii, local target: uncontrolled where the rank bit is set
                    if (r >> (cbit - boundary)) & 1:
                        pending[r].append(GateOp("single", op.gate, tbit))
                else:
                    pending[r].append(GateOp("controlled", op.gate, tbit, cbit))
            batch.append(pos)
            continue
        flush()
        if ds.scheme is None:
            raise ValidationError(f"qubit {tbit} requires communication but no scheme was configured")
        before_m, before_b = list(ds.messages_sent), list(ds.bytes_sent)
        t0 = time.perf_counter()
        if cbit is None:
            _exchange(ds, op.gate, tbit, ds.scheme)
        else:
            dist_apply_controlled(ds, op.gate, cbit, tbit)
        ds.sync()
        wall = time.perf_counter() - t0
        msgs = max(a - b for a, b in zip(ds.messages_sent, before_m))
        nbytes = max(a - b for a, b in zip(ds.bytes_sent, before_b))
        stats[pos] = GateStats(op.target, op.control, True, msgs, nbytes, wall)
        if norm_tol is not None:
            drift = abs(dist_norm2(ds) - 1.0)
            if drift > norm_tol:
                raise ValidationError(f"norm drifted by {drift:.3e} after gate {pos}")
    flush()
    return stats  # type: ignore[return-value]


def run_circuit(circuit: Circuit, plan: PartitionPlan, scheme: CommScheme | None = None,
                strat=None, transport: PeerTransport | None = None, execution: str = "cooperative",
                perm=None, kernel_backend: str | None = None, norm_tol: float | None = None, *,
                devices=None, initial=None, fused=False) -> tuple[DistState, list[GateStats]]:
    """engine.py:457-512 on the device, same positional order (circuit, plan,
    scheme, strat, transport, execution, perm, kernel_backend, norm_tol).
    Default: gate-by-gate with a device sync per gate so GateStats.wall_time
    means what it does in the reference.  fused=True (bit-identical) or
    "fast" (FMA + specialised passes): the local ops between global-target
    gates run as one fused svb_run_ops per rank, GateStats still per gate
    (_run_fused)."""
    if circuit.n != plan.n:
        raise ValidationError(f"circuit has {circuit.n} qubits, plan has {plan.n}")
    if perm is not None and perm.n != plan.n:
        raise ValidationError(f"layout is over {perm.n} qubits, plan has {plan.n}")
    ds = dist_init(plan, transport, scheme, execution, strat, kernel_backend, devices=devices, initial=initial)
    l2p = perm.logical_to_phys if perm is not None else tuple(range(plan.n))
    if fused:
        return ds, _run_fused(ds, circuit, l2p, norm_tol, fused == "fast")
    boundary = plan.n - plan.k
    stats: list[GateStats] = []
    for pos, op in enumerate(circuit.ops):
        tbit = l2p[op.target]
        before_m, before_b = list(ds.messages_sent), list(ds.bytes_sent)
        t0 = time.perf_counter()
        if op.kind == "single":
            if tbit < boundary:
                dist_apply_local(ds, op.gate, tbit)
            else:
                if ds.scheme is None:
                    raise ValidationError(f"qubit {tbit} requires communication but no scheme was configured")
                _exchange(ds, op.gate, tbit, ds.scheme)
        else:
            dist_apply_controlled(ds, op.gate, l2p[op.control], tbit)
        ds.sync()
        wall = time.perf_counter() - t0
        msgs = max(a - b for a, b in zip(ds.messages_sent, before_m))
        nbytes = max(a - b for a, b in zip(ds.bytes_sent, before_b))
        stats.append(GateStats(op.target, op.control, tbit >= boundary, msgs, nbytes, wall))
        if norm_tol is not None:
            drift = abs(dist_norm2(ds) - 1.0)
            if drift > norm_tol:
                raise ValidationError(f"norm drifted by {drift:.3e} after gate {pos}")
    return ds, stats


def time_ratio(comm, nocomm) -> float:
    """engine.py:515-521."""
    tc = comm.wall_time if isinstance(comm, GateStats) else float(comm)
    tn = nocomm.wall_time if isinstance(nocomm, GateStats) else float(nocomm)
    if tc <= 0.0 or tn <= 0.0:
        raise ValidationError("wall times must be positive to form a ratio")
    return tc / tn
