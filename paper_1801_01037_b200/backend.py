"""Kernel-backend module for the reference's plugin seam.

svsim resolves a backend name to a module exporting exactly two functions
(kernel/__init__.py:66-75; contract at _stride_py.py:93-98 and
_stride_cy.pyx:24-25, 57-58):

    apply_single(amps, q11, q12, q21, q22, target, mode, workers) -> None
    apply_controlled(amps, q11, q12, q21, q22, control, target, mode, workers) -> None

``amps`` is the caller-owned host complex128 array, updated in place; the
call is synchronous; mode/workers may be ignored (all reference modes are
bit-identical).  This module satisfies that contract with libsvb.so:
svb_host_apply_1q / svb_host_apply_c1q stream the array through HBM (64 MiB
units on three streams: copies in, kernel and copies out of different units
overlap; large arrays are page-locked once for full-duplex PCIe).  Registering it in svsim is a two-line change shown
in INTEGRATION.md.  Validation happens in the caller's wrapper, as in the
reference; the C layer re-checks and raises ValidationError on bad input.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .errors import ValidationError

NAME = "cuda"


def _q(q11, q12, q21, q22):
    vals = []
    for z in (q11, q12, q21, q22):
        z = complex(z)
        vals += [z.real, z.imag]
    return (ctypes.c_double * 8)(*vals)


# Large caller arrays are page-locked once (svb_host_register) so the
# streamed seam moves them at full-duplex PCIe speed; the registration is
# released when the array object is garbage-collected.
_PIN_MIN_BYTES = 4 << 20
_pinned: dict[tuple[int, int], weakref.finalize] = {}


def _unpin(key):
    _pinned.pop(key, None)
    try:
        _lib.load().svb_host_unregister(ctypes.c_void_p(key[0]))
    except Exception:  # interpreter teardown
        pass


def _pin(amps: np.ndarray) -> None:
    if amps.nbytes < _PIN_MIN_BYTES:
        return
    key = (amps.ctypes.data, amps.nbytes)
    if key in _pinned:
        return
    if _lib.load().svb_host_register(ctypes.c_void_p(key[0]), key[1]) == 0:
        _pinned[key] = weakref.finalize(amps, _unpin, key)


def _ptr(amps: np.ndarray) -> ctypes.c_void_p:
    if not isinstance(amps, np.ndarray) or amps.dtype != np.complex128 or not amps.flags.c_contiguous:
        raise ValidationError("backend operates on contiguous complex128 arrays")
    _pin(amps)
    return ctypes.c_void_p(amps.ctypes.data)


def apply_single(amps, q11, q12, q21, q22, target, mode, workers):
    lib = _lib.load()
    _lib.check(lib.svb_host_apply_1q(_ptr(amps), amps.shape[0], _q(q11, q12, q21, q22), int(target)),
               "apply_single")


def apply_controlled(amps, q11, q12, q21, q22, control, target, mode, workers):
    lib = _lib.load()
    _lib.check(lib.svb_host_apply_c1q(_ptr(amps), amps.shape[0], _q(q11, q12, q21, q22),
                                      int(control), int(target)), "apply_controlled")
