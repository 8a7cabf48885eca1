"""Multi-process partitioned engine: one process per GPU (torchrun / NCCL).

The reference runs 2^k ranks in one process over an in-memory FIFO
transport (engine.py:57-120, 279-341).  Here every rank is a process that
owns one GPU and one slab of L = 2^(n-k) amplitudes in HBM; torch.distributed
is the transport (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for tests).

Per op (engine.py:483-494):
* rank-local target: appended to a batch that runs as ONE fused
  svb_run_ops call (multi-gate HBM passes) when the next exchange is due;
* rank-bit target, non-diagonal gate: the paper's partner exchange with
  partner = rank ^ 2^(t-(n-k)) (partition.py:126-137), chunk-pipelined: the
  send/recv of chunk i+1 (torch.distributed P2P, NCCL's stream) overlaps the
  own-row update of chunk i (svb_exchange_own_row on the compute stream) --
  the own-row rule of scheme b (engine.py:249-254) in chunks of m
  amplitudes as in chunked(m) (engine.py:257-272), with no zero padding;
* local control + rank-bit target (regime ii, engine.py:444-447): only the
  control-set half is packed, exchanged and updated (8*L bytes each way);
* rank-bit control (regime iii, engine.py:432-443): only ranks with that bit
  set act; a local target then needs no communication at all;
* diagonal gate on a rank-bit target (Z S T Rz CP): no exchange -- every
  amplitude keeps its own row, scaled by q11 (bit clear) or q22 (bit set);
  ``elide_diagonal=False`` restores the reference's exchange for NVLink
  accounting (SURVEY 8(d) "diagonal-gate shortcut").

The compute backend is libsvb.so (CudaCompute).  Tests on CPU inject a
checker-backed compute object; the product never falls back to one.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np

from .core import Circuit, Gate2x2, GateOp
from .errors import ValidationError
from .partition import PartitionPlan

DEFAULT_CHUNK = 1 << 24  # amplitudes per pipelined message (256 MiB)


class CudaCompute:
    """libsvb.so kernels on this rank's GPU (torch owns buffers/streams)."""

    def __init__(self, device: int | None = None):
        import torch

        from . import _lib

        self.torch = torch
        self.lib = _lib.load()
        self._lib = _lib
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    def _sp(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def zeros(self, count: int):
        return self.torch.zeros(count, dtype=self.torch.complex128, device=self.device)

    def from_numpy(self, arr: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(arr)).to(self.device)

    def to_numpy(self, t) -> np.ndarray:
        return t.cpu().numpy()

    def run_ops(self, slab, ops, fuse: bool = True, strict: bool = False, fma: bool = False,
                jit: bool = False) -> None:
        if not ops:
            return
        arr, nops = self._lib.ops_array(ops if isinstance(ops, tuple) else tuple(ops))
        flags = self._lib.run_flags(fuse, strict, fma, jit)
        self._lib.check(self.lib.svb_run_ops(ctypes.c_void_p(slab.data_ptr()), slab.shape[0], arr,
                                             nops, flags, self._sp()), "run_ops")

    def pack_half(self, src, dst, count: int, bit: int, value: int, offset: int) -> None:
        self._lib.check(self.lib.svb_pack_half(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                               count, bit, value, offset, self._sp()), "pack_half")

    def unpack_half(self, dst, src, count: int, bit: int, value: int, offset: int) -> None:
        self._lib.check(self.lib.svb_unpack_half(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                                 count, bit, value, offset, self._sp()), "unpack_half")

    def pack(self, src, dst, count: int, cbit: int, offset: int) -> None:
        self._lib.check(self.lib.svb_pack_ctrl(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                               count, cbit, offset, self._sp()), "pack")

    def exchange_update(self, own, other, count: int, gate: Gate2x2, own_is_low: bool,
                        cbit: int, offset: int, own_offset: int = 0) -> None:
        """own-row update of `count` amplitudes; cbit >= 0: `other` is packed
        (control-set elements only) and offset is in packed index space."""
        q = self._lib.gate_array(gate)
        if cbit < 0:
            ptr = ctypes.c_void_p(own.data_ptr() + 16 * own_offset)
            self._lib.check(self.lib.svb_exchange_own_row(ptr, ctypes.c_void_p(other.data_ptr()), count, q,
                                                          int(own_is_low), -1, 0, self._sp()), "exchange")
        else:
            self._lib.check(self.lib.svb_exchange_own_row_packed(
                ctypes.c_void_p(own.data_ptr()), ctypes.c_void_p(other.data_ptr()), count, q,
                int(own_is_low), cbit, offset, self._sp()), "exchange")

    # -- peer-memory transport (DistEngine(peer=True)) --------------------

    def ipc_handle(self, slab) -> tuple[bytes, int]:
        """(handle of the allocation holding slab, slab's byte offset in it)"""
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        self._lib.check(self.lib.svb_ipc_handle(ctypes.c_void_p(slab.data_ptr()), h, ctypes.byref(off)),
                        "ipc_handle")
        return h.raw, off.value

    def ipc_open(self, handle: tuple[bytes, int]) -> tuple[int, int]:
        """(mapped allocation base, slab pointer)"""
        p = ctypes.c_void_p()
        self._lib.check(self.lib.svb_ipc_open(ctypes.c_char_p(handle[0]), ctypes.byref(p)), "ipc_open")
        return p.value, p.value + handle[1]

    def ipc_close(self, ptr: int) -> None:
        self._lib.check(self.lib.svb_ipc_close(ctypes.c_void_p(ptr)), "ipc_close")

    def pair_update(self, lo_ptr: int, hi_ptr: int, begin: int, end: int, gate: Gate2x2, cbit: int) -> None:
        self._lib.check(self.lib.svb_pair_update(ctypes.c_void_p(lo_ptr), ctypes.c_void_p(hi_ptr), begin, end,
                                                 self._lib.gate_array(gate), cbit, self._sp()), "pair_update")

    def peer_swap_half(self, a_ptr: int, b_ptr: int, begin: int, end: int, bit: int, va: int, vb: int) -> None:
        self._lib.check(self.lib.svb_peer_swap_half(ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), begin, end,
                                                    bit, va, vb, self._sp()), "peer_swap_half")

    def norm2(self, slab) -> float:
        out = ctypes.c_double()
        self._lib.check(self.lib.svb_norm2(ctypes.c_void_p(slab.data_ptr()), slab.shape[0],
                                           ctypes.byref(out), self._sp()), "norm2")
        return out.value

    def synchronize(self) -> None:
        self.torch.cuda.synchronize(self.device)


@dataclass
class ExchangeStats:
    exchanges: int = 0
    swaps: int = 0
    elided: int = 0
    bytes_sent: int = 0
    bytes_recv: int = 0
    messages: int = 0


def _is_diag(g: Gate2x2) -> bool:
    return complex(g.q12) == 0 and complex(g.q21) == 0


class DistEngine:
    """This process's rank of a 2^k-way partitioned n-qubit state."""

    def __init__(self, n: int, compute=None, group=None, initial=None, chunk: int = DEFAULT_CHUNK,
                 fuse: bool = True, elide_diagonal: bool = True, fma: bool = False, jit: bool = False,
                 layout: bool = False, peer: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        k = self.world.bit_length() - 1
        if (1 << k) != self.world:
            raise ValidationError(f"world size {self.world} is not a power of two")
        self.plan = PartitionPlan(n, k)
        self.n, self.k = n, k
        self.L = self.plan.local_len
        self.boundary = n - k
        self.compute = compute if compute is not None else CudaCompute()
        self.chunk = max(1, min(int(chunk), self.L))
        self.fuse = fuse
        self.fma, self.jit = fma, jit  # local segments: FMA fused passes / NVRTC-specialised
        # layout: run() swaps a global qubit into a local position (half-slab
        # exchange) when a non-diagonal gate targets it, instead of one
        # exchange per global gate; the identity layout is restored at the end
        self.layout = layout
        self.elide_diagonal = elide_diagonal
        self.stats = ExchangeStats()
        if initial is not None:
            amps = np.asarray(initial, np.complex128)
            if amps.shape[0] != (1 << n):
                raise ValidationError(f"initial state must have 2**{n} amplitudes")
            self.slab = self.compute.from_numpy(amps[self.rank * self.L:(self.rank + 1) * self.L])
        else:
            self.slab = self.compute.zeros(self.L)
            if self.rank == 0:
                self.slab[0] = 1.0
        self._pending: list[GateOp] = []
        self._pending_key = None  # the cached tuple _pending was copied from, if any
        self._scheds: dict = {}
        self._bufs = None
        # peer: exchanges and swaps read / write the partner's slab in place
        # (CUDA IPC; NVLink P2P between GPUs) -- one kernel per rank between
        # two barriers of the process group, which only carries control
        self.peer = peer
        self._peers: dict[int, int] = {}
        self._maps: list[int] = []
        if peer:
            # export (may fail, e.g. VMM-backed slabs under expandable_segments)
            # and import both report through the collectives below, so every
            # rank sees every failure and all fall back together -- none is
            # left waiting in a collective the others skipped
            mine, err = None, None
            try:
                mine = self.compute.ipc_handle(self.slab)
            except Exception as e:
                err = f"rank {self.rank}: export: {e}"
            handles = [None] * self.world
            dist.all_gather_object(handles, mine, group=self.group)
            if err is None and any(h is None for h in handles):
                err = "a partner could not export its slab"
            if err is None:
                try:
                    for r, h in enumerate(handles):
                        if r != self.rank:
                            base, ptr = self.compute.ipc_open(h)
                            self._maps.append(base)
                            self._peers[r] = ptr
                except Exception as e:  # e.g. no peer access between these GPUs
                    err = f"rank {self.rank}: import: {e}"
            errs = [None] * self.world
            dist.all_gather_object(errs, err, group=self.group)
            if any(errs):  # every rank falls back together to the send/recv transport
                for base in self._maps:
                    self.compute.ipc_close(base)
                self._peers, self._maps, self.peer = {}, [], False
                if self.rank == 0:
                    import sys

                    print(f"DistEngine: peer transport unavailable ({next(e for e in errs if e)}); "
                          "using send/recv", file=sys.stderr)

    def close(self) -> None:
        """Unmap the partners' slabs (peer mode); the engine is unusable after."""
        self.compute.synchronize()
        if self.peer:
            self.dist.barrier(group=self.group)
            for base in self._maps:
                self.compute.ipc_close(base)
            self._peers, self._maps = {}, []

    # -- helpers ------------------------------------------------------------

    def _buffers(self, count: int, packed: bool):
        m = min(self.chunk, count)
        if self._bufs is None or self._bufs[0].shape[0] < m:
            self._bufs = [self.compute.zeros(m) for _ in range(4)]  # recv x2, send x2
        return m

    def _flush(self) -> None:
        if self._pending:
            ops = self._pending_key if self._pending_key is not None else tuple(self._pending)
            if self.fma or self.jit:
                self.compute.run_ops(self.slab, ops, fuse=self.fuse, fma=self.fma, jit=self.jit)
            else:
                self.compute.run_ops(self.slab, ops, fuse=self.fuse)
            self._pending = []
        self._pending_key = None

    def _diag_local(self, g: Gate2x2, bit_set: bool, cbit: int | None) -> None:
        """Global-target diagonal gate: scale own amplitudes by q11 or q22."""
        s = complex(g.q22) if bit_set else complex(g.q11)
        if s == 1:
            return
        d = Gate2x2(s, 0, 0, s)
        if cbit is None:
            self._pending.append(GateOp("single", d, 0))
        else:
            self._pending.append(GateOp("controlled", d, 1 if cbit == 0 else 0, cbit))

    def _peer_sync(self) -> None:
        self.compute.synchronize()
        self.dist.barrier(group=self.group)

    def _exchange_peer(self, g: Gate2x2 | None, t: int, cbit: int | None) -> None:
        """Global-target gate over peer memory: the pair (mine[j], partner[j])
        is updated in place -- the lower rank for j < L/2, the upper for
        j >= L/2 (k_pair_update: 16*L bytes each way over the link, like a
        slab exchange, but no staging buffers and no separate update pass).  g None: this rank does not act (regime iii) but joins the
        barriers, which every rank passes twice per global gate."""
        self._flush()
        self._peer_sync()
        if g is not None:
            partner = self.rank ^ (1 << (t - self.boundary))
            low = self.rank < partner
            mine, theirs = self.slab.data_ptr(), self._peers[partner]
            lo, hi = (mine, theirs) if low else (theirs, mine)
            half = self.L // 2
            begin, end = (0, half) if low else (half, self.L)
            self.compute.pair_update(lo, hi, begin, end, g, -1 if cbit is None else cbit)
            count = self.L if cbit is None else self.L // 2
            self.stats.exchanges += 1
            self.stats.messages += 1
            # link bytes each way: my writes into the partner's half plus the
            # partner's reads of mine (the same 16 B per pair as send/recv,
            # without the staging copies)
            self.stats.bytes_sent += 16 * count
            self.stats.bytes_recv += 16 * count
        self._peer_sync()

    def _exchange(self, g: Gate2x2, t: int, cbit: int | None) -> None:
        if self.peer:
            return self._exchange_peer(g, t, cbit)
        self._flush()
        dist = self.dist
        partner = self.rank ^ (1 << (t - self.boundary))
        low = self.rank < partner
        count = self.L if cbit is None else self.L // 2
        m = self._buffers(count, cbit is not None)
        recv = self._bufs[0:2]
        send = self._bufs[2:4]
        nchunks = math.ceil(count / m)
        peer = dist.get_global_rank(self.group, partner) if self.group is not None else partner

        def post(ci):
            off = ci * m
            cnt = min(m, count - off)
            if cbit is None:
                src = self.slab[off:off + cnt]
            else:
                self.compute.pack(self.slab, send[ci % 2], cnt, cbit, off)
                src = send[ci % 2][:cnt]
            ops = [dist.P2POp(dist.isend, src, peer, self.group),
                   dist.P2POp(dist.irecv, recv[ci % 2][:cnt], peer, self.group)]
            return dist.batch_isend_irecv(ops)

        works = post(0)
        for ci in range(nchunks):
            nxt = post(ci + 1) if ci + 1 < nchunks else None
            for w in works:
                w.wait()
            off = ci * m
            cnt = min(m, count - off)
            if cbit is None:
                self.compute.exchange_update(self.slab, recv[ci % 2], cnt, g, low, -1, 0, own_offset=off)
            else:
                self.compute.exchange_update(self.slab, recv[ci % 2], cnt, g, low, cbit, off)
            works = nxt
        self.stats.exchanges += 1
        self.stats.messages += nchunks
        self.stats.bytes_sent += 16 * count
        self.stats.bytes_recv += 16 * count

    def _swap(self, g: int, l: int) -> None:
        """Swap rank bit (physical qubit) g with local bit l: each rank sends
        the half of its slab whose bit l differs from its own bit g to the
        partner and unpacks the partner's half into the same positions."""
        if self.peer:
            return self._swap_peer(g, l)
        self._flush()
        dist = self.dist
        partner = self.rank ^ (1 << (g - self.boundary))
        v = 1 - ((self.rank >> (g - self.boundary)) & 1)  # the half that leaves
        count = self.L // 2
        m = self._buffers(count, True)
        recv = self._bufs[0:2]
        send = self._bufs[2:4]
        nchunks = math.ceil(count / m)
        peer = dist.get_global_rank(self.group, partner) if self.group is not None else partner

        def post(ci):
            off = ci * m
            cnt = min(m, count - off)
            self.compute.pack_half(self.slab, send[ci % 2], cnt, l, v, off)
            ops = [dist.P2POp(dist.isend, send[ci % 2][:cnt], peer, self.group),
                   dist.P2POp(dist.irecv, recv[ci % 2][:cnt], peer, self.group)]
            return dist.batch_isend_irecv(ops)

        works = post(0)
        for ci in range(nchunks):
            nxt = post(ci + 1) if ci + 1 < nchunks else None
            for w in works:
                w.wait()
            off = ci * m
            cnt = min(m, count - off)
            self.compute.unpack_half(self.slab, recv[ci % 2], cnt, l, v, off)
            works = nxt
        self.stats.swaps += 1
        self.stats.messages += nchunks
        self.stats.bytes_sent += 16 * count
        self.stats.bytes_recv += 16 * count

    def _swap_peer(self, g: int, l: int) -> None:
        """Layout swap over peer memory: the half of my slab whose bit l is v
        trades places with the partner's half whose bit l is 1 - v, in place
        (k_peer_swap_half); the pair's two ranks split the L/2 positions."""
        self._flush()
        self._peer_sync()
        partner = self.rank ^ (1 << (g - self.boundary))
        v = 1 - ((self.rank >> (g - self.boundary)) & 1)  # the half that leaves
        quarter = self.L // 4
        begin, end = (0, quarter) if self.rank < partner else (quarter, self.L // 2)
        self.compute.peer_swap_half(self.slab.data_ptr(), self._peers[partner], begin, end, l, v, 1 - v)
        self.stats.swaps += 1
        self.stats.messages += 1
        self.stats.bytes_sent += 16 * (self.L // 2)
        self.stats.bytes_recv += 16 * (self.L // 2)
        self._peer_sync()

    def _schedule_layout(self, ops: tuple) -> tuple[list, int]:
        """Action list with dynamic global<->local qubit swaps.
        The layout is kept as disjoint transpositions (global home position
        <-> local home position): a non-diagonal gate on a qubit that sits at
        a rank bit first swaps it with the local qubit whose next use as a
        non-diagonal target is farthest away (Belady), or swaps back a local
        qubit that was parked there.  Gates then address physical positions;
        the transpositions are undone at the end."""
        n, b = self.n, self.boundary
        pi = list(range(n))   # logical -> physical
        inv = list(range(n))  # physical -> logical
        uses = [[] for _ in range(n)]  # op indices where a qubit is a non-diagonal target
        for i, op in enumerate(ops):
            if not _is_diag(op.gate):
                uses[op.target].append(i)
        ptr = [0] * n
        actions, pending = [], []
        elided = 0

        def flush():
            if pending:
                actions.append(("local", tuple(pending)))
                pending.clear()

        def swap(gp, lp):
            flush()
            actions.append(("swap", gp, lp))
            qg, ql = inv[gp], inv[lp]
            pi[qg], pi[ql] = lp, gp
            inv[gp], inv[lp] = ql, qg

        def next_use(q, i):
            u = uses[q]
            while ptr[q] < len(u) and u[ptr[q]] < i:
                ptr[q] += 1
            return u[ptr[q]] if ptr[q] < len(u) else len(ops) + 1

        for i, op in enumerate(ops):
            g = op.gate
            t = pi[op.target]
            c = pi[op.control] if op.control is not None else None
            if t >= b and not (self.elide_diagonal and _is_diag(g)):
                if inv[t] >= b:  # a global qubit at home: park a local one there
                    best, far = -1, -1
                    for lp in range(b):
                        q = inv[lp]
                        if q != lp or lp == c:  # keep transpositions disjoint; keep the control local
                            continue
                        nu = next_use(q, i)
                        if nu > far:
                            best, far = lp, nu
                    swap(t, best)
                else:  # a parked local qubit p = inv[t]: swap it back to its home p
                    swap(t, inv[t])
                t = pi[op.target]
                c = pi[op.control] if op.control is not None else None
            if c is not None and c >= b:
                if not (self.rank >> (c - b)) & 1:
                    continue
                c = None
            if t < b:
                pending.append(GateOp("single", g, t) if c is None else GateOp("controlled", g, t, c))
                continue
            bit_set = bool((self.rank >> (t - b)) & 1)  # diagonal on a rank bit: a local phase
            s_ = complex(g.q22) if bit_set else complex(g.q11)
            elided += 1
            if s_ != 1:
                d = Gate2x2(s_, 0, 0, s_)
                pending.append(GateOp("single", d, 0) if c is None else
                               GateOp("controlled", d, 1 if c == 0 else 0, c))
        for gp in range(b, n):  # undo the parked transpositions
            if inv[gp] != gp:
                swap(gp, pi[gp])
        flush()
        return actions, elided

    # -- public ---------------------------------------------------------------

    def apply(self, op: GateOp) -> None:
        """One op with the reference's regime dispatch (engine.py:488-494, 415-450)."""
        t, c, g = op.target, op.control, op.gate
        b = self.boundary
        if c is not None and c >= b:
            if not (self.rank >> (c - b)) & 1:
                # regime (iii): this rank's control bit is clear; over peer
                # memory it still joins the exchange's barriers
                if self.peer and t >= b and not (self.elide_diagonal and _is_diag(g)):
                    self._exchange(None, t, None)
                return
            c = None  # acts as an uncontrolled gate on participating ranks
        if t < b:
            self._pending.append(GateOp("single", g, t) if c is None else GateOp("controlled", g, t, c))
            return
        bit_set = bool((self.rank >> (t - b)) & 1)
        if self.elide_diagonal and _is_diag(g):
            self._diag_local(g, bit_set, c)
            self.stats.elided += 1
            return
        self._exchange(g, t, c)

    def _schedule(self, ops: tuple) -> tuple[list, int]:
        """This rank's action list for an op tuple -- ("local", op tuple) runs
        and ("exchange", gate, target, control) steps -- as apply() would
        produce it; cached per circuit so repeated runs do no per-op Python
        work (the local tuples also hit the packed-op cache)."""
        hit = self._scheds.get(id(ops))
        if hit is not None and hit[0] is ops:
            return hit[1], hit[2]
        if self.layout:
            actions, elided = self._schedule_layout(ops)
            if len(self._scheds) >= 8:
                self._scheds.pop(next(iter(self._scheds)))
            self._scheds[id(ops)] = (ops, actions, elided)
            return actions, elided
        saved, self._pending = self._pending, []
        actions, elided = [], 0
        exchange = self._exchange
        try:
            def record(g, t, c):
                if self._pending:
                    actions.append(("local", tuple(self._pending)))
                    self._pending = []
                actions.append(("exchange", g, t, c))
            self._exchange = record
            before = self.stats.elided
            for op in ops:
                self.apply(op)
            elided = self.stats.elided - before
            self.stats.elided = before
            if self._pending:
                actions.append(("local", tuple(self._pending)))
        finally:
            self._exchange = exchange
            self._pending = saved
        if len(self._scheds) >= 8:
            self._scheds.pop(next(iter(self._scheds)))
        self._scheds[id(ops)] = (ops, actions, elided)
        return actions, elided

    def run(self, circuit: Circuit) -> "DistEngine":
        if circuit.n != self.n:
            raise ValidationError(f"circuit has {circuit.n} qubits, engine has {self.n}")
        self._flush()
        actions, elided = self._schedule(circuit.ops)
        for act in actions:
            if act[0] == "local":
                self._pending = list(act[1])
                self._pending_key = act[1]
                self._flush()
            elif act[0] == "swap":
                self._swap(act[1], act[2])
            else:
                self._exchange(act[1], act[2], act[3])
        self.stats.elided += elided
        return self

    def norm2(self) -> float:
        import torch

        self._flush()
        local = self.compute.norm2(self.slab)
        t = torch.tensor([local], dtype=torch.float64, device=self._coll_device())
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    def _coll_device(self):
        import torch

        nccl = self.dist.get_backend(self.group) == "nccl"
        return self.slab.device if (nccl and self.slab.is_cuda) else torch.device("cpu")

    def gather(self) -> np.ndarray | None:
        """Full state on rank 0 (engine.py:188-192); None elsewhere."""
        import torch

        self._flush()
        dev = self._coll_device()
        mine = self.slab.to(dev)
        parts = [torch.zeros(self.L, dtype=torch.complex128, device=dev) for _ in range(self.world)]
        self.dist.all_gather(parts, mine, group=self.group)
        if self.rank != 0:
            return None
        return np.concatenate([p.cpu().numpy() for p in parts])


# ---------------------------------------------------------------------------
# bench.py --gpus N (torchrun): weak scaling, 2^26 amplitudes per GPU


def bench_main(args, clock_cls=None, peaks_fn=None) -> None:
    """bench.py's N>1 arm (and SVB_BENCH_DIST=1 at world 1).  clock_cls /
    peaks_fn: bench.py's nvidia-smi sampler and measured-peak reader."""
    import contextlib
    import json
    import time

    import torch
    import torch.distributed as dist

    from . import _lib, workloads

    # one GPU per rank; SVB_DIST_BACKEND=gloo (control plane on the host,
    # ranks may share a GPU) is a functional smoke of this path on one GPU
    # with the peer transport -- its timings are not a multi-GPU measurement
    backend = os.environ.get("SVB_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"
    rank, world = dist.get_rank(), dist.get_world_size()
    k = world.bit_length() - 1
    n = 26 + k
    layers = int(os.environ.get("SVB_BENCH_LAYERS", "200"))
    circuit = workloads.random_layer_circuit(n, layers)
    nops = len(circuit.ops)
    eng = DistEngine(n, fma=getattr(args, "fma", True), jit=getattr(args, "jit", True),
                     layout=os.environ.get("SVB_DIST_LAYOUT", "1") != "0",
                     peer=os.environ.get("SVB_DIST_PEER", "1") != "0" and world > 1)
    stream = torch.cuda.current_stream()

    def step():
        eng.slab.zero_()
        if rank == 0:
            eng.slab[0] = 1.0
        eng.run(circuit)

    for _ in range(max(args.warmup, 0)):
        step()
    launches0 = _lib.launch_count()
    stats0 = (eng.stats.exchanges, eng.stats.bytes_sent, eng.stats.swaps)
    dist.barrier()
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = clock_cls(local) if (clock_cls and rank == 0) else contextlib.nullcontext()
    with sampler as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    launches = _lib.launch_count() - launches0
    stats1 = (eng.stats.exchanges, eng.stats.bytes_sent, eng.stats.swaps)  # the timed steps only
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    norm = eng.norm2()

    # e2e: every rank copies its slab in from pinned host memory, runs the
    # circuit, copies the slab back out; max wall time over ranks
    slab_bytes = eng.slab.numel() * 16
    host_in = torch.zeros(eng.slab.numel(), dtype=torch.complex128).pin_memory()
    if rank == 0:
        host_in[0] = 1.0
    host_out = torch.empty_like(host_in).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.slab.copy_(host_in, non_blocking=True)
        eng.run(circuit)
        host_out.copy_(eng.slab, non_blocking=True)
        torch.cuda.synchronize()
    e2e_dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
    dist.all_reduce(e2e_dt, op=dist.ReduceOp.MAX)
    e2e_dt = float(e2e_dt.item())
    if rank == 0:
        ex = stats1[0] - stats0[0]
        sent = stats1[1] - stats0[1]
        line = {
            "metric": "gate applications/s", "value": round(nops * args.steps / (ms / 1e3), 1),
            "unit": "gate_apps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded circuit, |0...0>)",
            "config": {"workload": f"random layer circuit n={n} ({layers} layers) over {world} GPUs, "
                                   f"2^26 amplitudes per GPU, {k} global qubits",
                       "n_qubits": n, "global_qubits": k, "parallelism": f"state partition x{world}"},
            "transport": "peer memory (CUDA IPC, one kernel per rank per exchange / swap)" if eng.peer
                         else "NCCL send/recv, chunk-pipelined",
            "exchanges_per_step": ex / args.steps,
            "layout_swaps_per_step": (stats1[2] - stats0[2]) / args.steps,
            "nvlink_bytes_sent_per_gpu_per_step": sent / args.steps,
            "gpu_launches": launches,
            "e2e": {"value": round(nops * e2e_steps / e2e_dt, 1), "unit": "gate_apps/s",
                    "h2d_bytes_per_step": world * slab_bytes, "d2h_bytes_per_step": world * slab_bytes,
                    "api": "DistEngine.run on each rank's slab, pinned H2D + run + D2H per step",
                    "steps": e2e_steps},
            "check": {"norm": norm},
        }
        if prof:
            name, (cnt, tms, nbytes) = max(prof.items(), key=lambda kv: kv[1][1])
            peak, peak_src = peaks_fn() if peaks_fn else (6650.0, "fallback")
            achieved = nbytes / (tms / 1e3) / 1e9
            line["roofline"] = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 1), "peak": peak,
                                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                                "avg_launch_ms": round(tms / cnt, 4), "launches": cnt,
                                "share_of_step": round(tms / ms, 4), "peak_source": peak_src,
                                "rank": 0}
        if clock_cls:
            line["clocks"] = clk.summary()
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
