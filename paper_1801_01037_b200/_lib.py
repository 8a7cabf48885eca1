"""ctypes binding of libsvb.so (include/svb.h).

This is exactly the stub a maintainer would add on the reference side
(INTEGRATION.md): plain pointers, sizes and 8-double gate records.  There is
no fallback -- if the library is missing or no CUDA device is visible, every
compute entry point raises NativeLibraryMissing / SvsimError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (
    CapacityError,
    ContractViolation,
    NativeLibraryMissing,
    SvsimError,
    ValidationError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVB_LIB") or os.path.join(HERE, "libsvb.so")

SVB_OK, SVB_EINVAL, SVB_ENOMEM, SVB_ECUDA, SVB_ENCCL, SVB_ESTATE = 0, -1, -2, -3, -4, -5
RUN_FUSE = 1
RUN_STRICT_ORDER = 2
RUN_FMA = 4
RUN_JIT = 8
RUN_JIT_ASYNC = 16


def run_flags(fuse: bool = True, strict_order: bool = False, fma: bool = False, jit=False) -> int:
    """jit: False, True (compile on first use, synchronously) or "async"
    (interpreter until the background compile finishes)."""
    return ((RUN_FUSE if fuse else 0) | (RUN_STRICT_ORDER if strict_order else 0)
            | (RUN_FMA if fma else 0) | (RUN_JIT if jit else 0)
            | (RUN_JIT_ASYNC if jit == "async" else 0))

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p


class SvbOp(ctypes.Structure):
    """svb_op (include/svb.h) -- one GateOp (core.py:97-115)."""

    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32),
                ("control", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("q", ctypes.c_double * 8)]


_SIGS = {
    "svb_abi_version": ([], _int),
    "svb_last_error": ([], ctypes.c_char_p),
    "svb_launch_count": ([], _i64),
    "svb_apply_1q": ([_vp, _i64, _dp, _int, _vp], _int),
    "svb_apply_c1q": ([_vp, _i64, _dp, _int, _int, _vp], _int),
    "svb_run_ops": ([_vp, _i64, ctypes.POINTER(SvbOp), _int, ctypes.c_uint, _vp], _int),
    "svb_plan_passes": ([_int, ctypes.POINTER(SvbOp), _int, ctypes.c_uint, ctypes.POINTER(_int),
                         ctypes.POINTER(_int)], _int),
    "svb_swap_suffix": ([_int, ctypes.POINTER(SvbOp), _int], _int),
    "svb_jit_check": ([_int, ctypes.POINTER(SvbOp), _int, ctypes.c_uint, ctypes.POINTER(_int)], _int),
    "svb_jit_counters": ([ctypes.POINTER(ctypes.c_long), ctypes.POINTER(ctypes.c_long)], None),
    "svb_jit_wait": ([], None),
    "svb_stream_signal": ([_vp, ctypes.c_uint32, _vp], _int),
    "svb_stream_wait": ([_vp, ctypes.c_uint32, _vp], _int),
    "svb_peer_copy": ([_vp, _vp, _i64, _vp], _int),
    "svb_copy_async": ([_vp, _vp, _i64, _vp], _int),
    "svb_host_register": ([_vp, _i64], _int),
    "svb_host_unregister": ([_vp], _int),
    "svb_norm2": ([_vp, _i64, _dp, _vp], _int),
    "svb_probs": ([_vp, _i64, _vp, _vp], _int),
    "svb_dense_embed": ([_vp, _int, _dp, _int, _int, _vp], _int),
    "svb_dense_matvec": ([_vp, _vp, _vp, _i64, _i64, _i64, _vp], _int),
    "svb_exchange_own_row": ([_vp, _vp, _i64, _dp, _int, _int, _i64, _vp], _int),
    "svb_pair_update": ([_vp, _vp, _i64, _i64, _dp, _int, _vp], _int),
    "svb_pack_ctrl": ([_vp, _vp, _i64, _int, _i64, _vp], _int),
    "svb_pack_half": ([_vp, _vp, _i64, _int, _int, _i64, _vp], _int),
    "svb_unpack_half": ([_vp, _vp, _i64, _int, _int, _i64, _vp], _int),
    "svb_permute_qubits": ([_vp, _vp, _i64, ctypes.POINTER(_int), _int, _vp], _int),
    "svb_exchange_own_row_packed": ([_vp, _vp, _i64, _dp, _int, _int, _i64, _vp], _int),
    "svb_host_apply_1q": ([_vp, _i64, _dp, _int], _int),
    "svb_host_apply_c1q": ([_vp, _i64, _dp, _int, _int], _int),
    "svb_host_run_ops": ([_vp, _vp, _i64, ctypes.POINTER(SvbOp), _int, ctypes.c_uint], _int),
    "svb_release_staging": ([], _int),
    "svb_peer_swap_half": ([_vp, _vp, _i64, _i64, _int, _int, _int, _vp], _int),
    "svb_ipc_handle": ([_vp, ctypes.c_char_p, ctypes.POINTER(_i64)], _int),
    "svb_ipc_open": ([ctypes.c_char_p, ctypes.POINTER(_vp)], _int),
    "svb_ipc_close": ([_vp], _int),
    "svb_host_run_ops_batch": ([ctypes.POINTER(_vp), ctypes.POINTER(_vp), _int, _i64, ctypes.POINTER(SvbOp), _int,
                                ctypes.c_uint], _int),
    "svb_profile_enable": ([_int], _int),
    "svb_profile_read": ([_int, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)], _int),
    "svb_profile_class_name": ([_int], ctypes.c_char_p),
    "svb_dist_create": ([_int, _int, ctypes.POINTER(_int), ctypes.POINTER(_vp), ctypes.POINTER(_vp)], _int),
    "svb_dist_apply_1q": ([_vp, _dp, _int], _int),
    "svb_dist_apply_c1q": ([_vp, _dp, _int, _int], _int),
    "svb_dist_norm2": ([_vp, _dp], _int),
    "svb_dist_stats": ([_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)], _int),
    "svb_dist_sync": ([_vp], _int),
    "svb_dist_destroy": ([_vp], _int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(require_cuda: bool = True):
    """Load libsvb.so.  Raises NativeLibraryMissing if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise NativeLibraryMissing("no CUDA device visible; the gate engine is GPU-only")
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == SVB_OK:
        return
    msg = (_lib.svb_last_error() or b"").decode(errors="replace")
    msg = f"{what}: {msg}" if what else msg
    if rc == SVB_EINVAL:
        raise ValidationError(msg)
    if rc == SVB_ENOMEM:
        raise CapacityError(msg)
    if rc == SVB_ESTATE:
        raise ContractViolation(msg)
    raise SvsimError(f"{msg} (svb status {rc})")


def gate_array(g) -> ctypes.Array:
    """Gate2x2 / 4 complex / 8 doubles -> ctypes double[8]."""
    if hasattr(g, "as_doubles"):
        vals = g.as_doubles()
    elif hasattr(g, "q11"):
        vals = [v for z in (g.q11, g.q12, g.q21, g.q22) for v in (complex(z).real, complex(z).imag)]
    else:
        arr = np.asarray(g)
        if arr.dtype.kind == "c":
            arr = arr.reshape(-1)
            vals = [v for z in arr for v in (z.real, z.imag)]
        else:
            vals = [float(v) for v in arr.reshape(-1)]
    if len(vals) != 8:
        raise ValidationError("gate must have four complex entries")
    return (ctypes.c_double * 8)(*vals)


_OP_DTYPE = np.dtype([("kind", "<i4"), ("target", "<i4"), ("control", "<i4"), ("reserved", "<i4"),
                      ("q", "<f8", (8,))])
assert _OP_DTYPE.itemsize == ctypes.sizeof(SvbOp)
_OPS_CACHE: dict = {}  # id(ops tuple) -> (the tuple, packed array, count); recent circuits / segments


def ops_array(ops) -> tuple[ctypes.Array, int]:
    """Iterable of GateOp -> svb_op[].  Packing is vectorised, and the packed
    array of an (immutable) op tuple is cached, so calling the same circuit
    again -- bench steps, parameter sweeps -- costs no per-op Python work."""
    key = id(ops) if isinstance(ops, tuple) else None
    if key is not None:
        hit = _OPS_CACHE.get(key)
        if hit is not None and hit[0] is ops:
            return hit[1], hit[2]
    seq = list(ops)
    n = len(seq)
    packed = np.zeros(max(n, 1), dtype=_OP_DTYPE)
    if n:
        packed["kind"][:n] = [0 if op.kind == "single" else 1 for op in seq]
        packed["target"][:n] = [int(op.target) for op in seq]
        packed["control"][:n] = [-1 if op.control is None else int(op.control) for op in seq]
        packed["q"][:n] = [op.gate.as_doubles() for op in seq]
    arr = (SvbOp * max(n, 1)).from_buffer(packed)
    if key is not None:
        if len(_OPS_CACHE) >= 512:
            _OPS_CACHE.pop(next(iter(_OPS_CACHE)))
        _OPS_CACHE[key] = (ops, arr, n)
    return arr, n


PROFILE_CLASSES = ("k_pair_high", "k_pair_low", "k_diag", "k_tiny", "k_fused", "k_exchange", "k_norm",
                   "kpass_jit", "k_dense")


def profile_enable(on: bool = True) -> None:
    check(load().svb_profile_enable(1 if on else 0), "profile_enable")


def profile_read() -> dict:
    """{class name: (launches, total_ms, algorithmic bytes)} since enable."""
    lib = load()
    out = {}
    for cls, name in enumerate(PROFILE_CLASSES):
        n, ms, b = _i64(), ctypes.c_double(), _i64()
        check(lib.svb_profile_read(cls, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b)), "profile_read")
        if n.value:
            out[name] = (n.value, ms.value, b.value)
    return out


def launch_count() -> int:
    return int(load(require_cuda=False).svb_launch_count())


def jit_counters() -> tuple[int, int]:
    """(cubins read from the on-disk JIT cache, NVRTC compiles) since load."""
    hits, comps = ctypes.c_long(), ctypes.c_long()
    load(require_cuda=False).svb_jit_counters(ctypes.byref(hits), ctypes.byref(comps))
    return hits.value, comps.value


def jit_wait() -> None:
    """Wait for background pass compiles (run_flags(jit="async"))."""
    load(require_cuda=False).svb_jit_wait()
