"""Device-resident state vectors and the calls that act on them.

PyTorch owns the HBM buffer (a complex128 CUDA tensor = interleaved double2)
and supplies the stream; every computation is a libsvb.so kernel reached
through the C ABI.  Calls are stream-ordered on torch's current stream, so
they compose with torch code without extra synchronisation.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .core import Circuit, Gate2x2, GateOp, StateVector
from .errors import CapacityError, ValidationError


def _torch():
    import torch

    return torch


def _stream_ptr():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class DeviceState:
    """n-qubit state in HBM: ``amps`` is a contiguous complex128 CUDA tensor."""

    __slots__ = ("n", "amps")

    def __init__(self, n: int, amps):
        torch = _torch()
        if not isinstance(amps, torch.Tensor) or amps.dtype != torch.complex128 or not amps.is_cuda:
            raise ValidationError("DeviceState needs a complex128 CUDA tensor")
        if amps.dim() != 1 or amps.shape[0] != (1 << n) or not amps.is_contiguous():
            raise ValidationError(f"amplitude tensor must be contiguous with length 2**{n}")
        self.n = int(n)
        self.amps = amps

    @classmethod
    def zeros(cls, n: int, device=None) -> "DeviceState":
        """|0...0> (core.py:148-154) without the host-side MAX_QUBITS cap:
        the cap here is HBM (2^33 amplitudes = 128 GiB fits one B200)."""
        torch = _torch()
        _lib.load()
        if n < 1 or n > 36:
            raise CapacityError(f"qubit count {n} outside [1, 36]")
        try:
            amps = torch.zeros(1 << n, dtype=torch.complex128, device=device or "cuda")
        except torch.OutOfMemoryError as exc:
            raise CapacityError(f"2^{n} amplitudes do not fit in device memory") from exc
        amps[0] = 1.0
        return cls(n, amps)

    @classmethod
    def from_host(cls, s, device=None) -> "DeviceState":
        torch = _torch()
        _lib.load()
        arr = s.amps if isinstance(s, StateVector) else np.ascontiguousarray(s, np.complex128)
        n = int(arr.shape[0]).bit_length() - 1
        if arr.shape[0] != (1 << n):
            raise ValidationError("amplitude count must be a power of two")
        return cls(n, torch.from_numpy(arr).to(device or "cuda"))

    @classmethod
    def random(cls, n: int, seed: int, device=None) -> "DeviceState":
        """Seeded normalized complex Gaussian generated in HBM (SURVEY 8(d):
        states too large for a host copy are made on the device)."""
        torch = _torch()
        _lib.load()
        gen = torch.Generator(device=device or "cuda")
        gen.manual_seed(seed)
        amps = torch.empty(1 << n, dtype=torch.complex128, device=device or "cuda")
        amps.view(torch.float64).normal_(generator=gen)
        st = cls(n, amps)
        amps.mul_(1.0 / np.sqrt(norm2(st)))
        return st

    def to_host(self) -> StateVector:
        return StateVector(self.n, self.amps.cpu().numpy(), validate=False)

    @property
    def ptr(self) -> ctypes.c_void_p:
        return ctypes.c_void_p(self.amps.data_ptr())

    def __len__(self) -> int:
        return 1 << self.n


def _as_device(s) -> tuple[ctypes.c_void_p, int]:
    torch = _torch()
    if isinstance(s, DeviceState):
        return s.ptr, 1 << s.n
    if isinstance(s, torch.Tensor):
        if s.dtype != torch.complex128 or not s.is_cuda or not s.is_contiguous():
            raise ValidationError("kernel operates on contiguous complex128 CUDA tensors")
        return ctypes.c_void_p(s.data_ptr()), int(s.shape[0])
    raise ValidationError("expected a DeviceState or a complex128 CUDA tensor")


def apply_single(s, g: Gate2x2, i: int):
    """In-place gate on qubit i (kernel/__init__.py:107-117), device buffer."""
    lib = _lib.load()
    ptr, n_amps = _as_device(s)
    _lib.check(lib.svb_apply_1q(ptr, n_amps, _lib.gate_array(g), int(i), _stream_ptr()),
               "apply_single")
    return s


def apply_controlled(s, g: Gate2x2, c: int, t: int):
    """In-place gate on t where bit c is set (kernel/__init__.py:120-134)."""
    lib = _lib.load()
    ptr, n_amps = _as_device(s)
    _lib.check(lib.svb_apply_c1q(ptr, n_amps, _lib.gate_array(g), int(c), int(t), _stream_ptr()),
               "apply_controlled")
    return s


def run_ops(s, ops, fuse: bool = True, strict_order: bool = False, fma: bool = False, jit: bool = False):
    """Apply ops in circuit order on the device (one rank of run_circuit,
    engine.py:483-494), optionally fused into shared-memory passes
    (strict_order: bit-identical to op-by-op; fma: fused passes contract
    multiply-adds, ~1 ulp from the reference; jit: fused passes compiled to
    straight-line kernels once per op list, same bits as the interpreter)."""
    lib = _lib.load()
    ptr, n_amps = _as_device(s)
    if isinstance(ops, Circuit):
        ops = ops.ops
    arr, nops = _lib.ops_array(ops)
    flags = _lib.run_flags(fuse, strict_order, fma, jit)
    _lib.check(lib.svb_run_ops(ptr, n_amps, arr, nops, flags, _stream_ptr()), "run_ops")
    return s


def plan_stats(n: int, ops, fuse: bool = True, strict_order: bool = False,
               jit: bool = False) -> tuple[int, int]:
    """(HBM passes, shared-memory register groups) the planner makes (host
    only); jit: the plan runtime-specialised passes get (larger tiles)."""
    lib = _lib.load(require_cuda=False)
    if isinstance(ops, Circuit):
        ops = ops.ops
    arr, nops = _lib.ops_array(ops)
    flags = _lib.run_flags(fuse, strict_order, jit=jit)
    out, groups = ctypes.c_int(0), ctypes.c_int(0)
    _lib.check(lib.svb_plan_passes(int(n), arr, nops, flags, ctypes.byref(out), ctypes.byref(groups)),
               "plan_passes")
    return out.value, groups.value


def plan_passes(n: int, ops, fuse: bool = True, strict_order: bool = False, jit: bool = False) -> int:
    return plan_stats(n, ops, fuse, strict_order, jit)[0]


def norm2(s) -> float:
    """sum |a|^2 on the device (core.py:171-174); synchronises the stream."""
    lib = _lib.load()
    ptr, n_amps = _as_device(s)
    out = ctypes.c_double(0.0)
    _lib.check(lib.svb_norm2(ptr, n_amps, ctypes.byref(out), _stream_ptr()), "norm2")
    return out.value


def probs(s):
    """|a_j|^2 as a float64 CUDA tensor (the measured-probability vector)."""
    torch = _torch()
    lib = _lib.load()
    ptr, n_amps = _as_device(s)
    dev = s.amps.device if isinstance(s, DeviceState) else s.device
    out = torch.empty(n_amps, dtype=torch.float64, device=dev)
    _lib.check(lib.svb_probs(ptr, n_amps, ctypes.c_void_p(out.data_ptr()), _stream_ptr()), "probs")
    return out


def _host_c128(a, writable: bool = False) -> np.ndarray:
    if isinstance(a, StateVector):
        a = a.amps
    ok = (isinstance(a, np.ndarray) and a.dtype == np.complex128 and a.flags.c_contiguous
          and (a.flags.writeable or not writable))
    return a if ok else np.ascontiguousarray(a, np.complex128).copy()


def simulate(circuit: Circuit, initial=None, fuse: bool = True, strict_order: bool = False,
             out: np.ndarray | None = None, fma: bool = False, jit: bool = False) -> np.ndarray:
    """End-to-end public call on HOST memory: copy the initial state (default
    |0...0>) to the device, run the whole circuit, copy the result back into
    `out` (default: `initial` itself when it is a writable complex128 array,
    else a new array).  Goes through svb_host_run_ops (include/svb.h);
    pinned host buffers get full PCIe bandwidth."""
    lib = _lib.load()
    if initial is None:
        src = np.zeros(1 << circuit.n, np.complex128)
        src[0] = 1.0
    else:
        src = _host_c128(initial, writable=out is None)
    if src.shape[0] != (1 << circuit.n):
        raise ValidationError(f"initial state has {src.shape[0]} amplitudes, circuit needs 2**{circuit.n}")
    dst = src if out is None else out
    if not (isinstance(dst, np.ndarray) and dst.dtype == np.complex128 and dst.flags.c_contiguous
            and dst.flags.writeable and dst.shape == src.shape):
        raise ValidationError("out must be a writable contiguous complex128 array of the state's size")
    arr, nops = _lib.ops_array(circuit.ops)
    flags = _lib.run_flags(fuse, strict_order, fma, jit)
    _lib.check(lib.svb_host_run_ops(ctypes.c_void_p(src.ctypes.data), ctypes.c_void_p(dst.ctypes.data),
                                    src.shape[0], arr, nops, flags), "simulate")
    return dst


def simulate_batch(circuit: Circuit, inputs, outs=None, fuse: bool = True, strict_order: bool = False,
                   fma: bool = False, jit: bool = False) -> list:
    """`simulate` over a batch of host states (one circuit, many inputs):
    through svb_host_run_ops_batch, which overlaps the H2D copy of the next
    state and the D2H copy of the previous one with the current run.
    outs[k] (default: inputs[k], in place) receives state k's result, bit
    for bit what simulate would return.  Use pinned buffers for overlap."""
    lib = _lib.load()
    size = 1 << circuit.n
    srcs = [_host_c128(x, writable=outs is None) for x in inputs]
    dsts = srcs if outs is None else list(outs)
    if len(dsts) != len(srcs):
        raise ValidationError(f"{len(srcs)} inputs but {len(dsts)} outputs")
    for x, y in zip(srcs, dsts):
        if x.shape[0] != size:
            raise ValidationError(f"initial state has {x.shape[0]} amplitudes, circuit needs 2**{circuit.n}")
        if not (isinstance(y, np.ndarray) and y.dtype == np.complex128 and y.flags.c_contiguous
                and y.flags.writeable and y.shape == x.shape):
            raise ValidationError("outs must be writable contiguous complex128 arrays of the state's size")
    arr, nops = _lib.ops_array(circuit.ops)
    flags = _lib.run_flags(fuse, strict_order, fma, jit)
    pin = (ctypes.c_void_p * max(1, len(srcs)))(*[x.ctypes.data for x in srcs])
    pout = (ctypes.c_void_p * max(1, len(dsts)))(*[y.ctypes.data for y in dsts])
    _lib.check(lib.svb_host_run_ops_batch(pin, pout, len(srcs), size, arr, nops, flags), "simulate_batch")
    return dsts


def release_staging() -> None:
    """Free the device buffers simulate / simulate_batch keep between calls."""
    _lib.check(_lib.load().svb_release_staging(), "release_staging")


def gate_op(kind: str, gate: Gate2x2, target: int, control: int | None = None) -> GateOp:
    return GateOp(kind, gate, target, control)
