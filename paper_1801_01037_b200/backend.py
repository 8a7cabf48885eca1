"""Kernel-backend module for the reference's plugin seam.

svsim resolves a backend name to a module exporting exactly two functions
(kernel/__init__.py:66-75; contract at _stride_py.py:93-98 and
_stride_cy.pyx:24-25, 57-58):

    apply_single(amps, q11, q12, q21, q22, target, mode, workers) -> None
    apply_controlled(amps, q11, q12, q21, q22, control, target, mode, workers) -> None

``amps`` is the caller-owned host complex128 array, updated in place; the
call is synchronous; mode/workers may be ignored (all reference modes are
bit-identical).  This module satisfies that contract with libsvb.so:
svb_host_apply_1q / svb_host_apply_c1q copy the array to HBM, run one
kernel and copy it back.  Registering it in svsim is a two-line change shown
in INTEGRATION.md.  Validation happens in the caller's wrapper, as in the
reference; the C layer re-checks and raises ValidationError on bad input.
"""

from __future__ import annotations

import ctypes

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


def _ptr(amps: np.ndarray) -> ctypes.c_void_p:
    if not isinstance(amps, np.ndarray) or amps.dtype != np.complex128 or not amps.flags.c_contiguous:
        raise ValidationError("backend operates on contiguous complex128 arrays")
    return ctypes.c_void_p(amps.ctypes.data)


def apply_single(amps, q11, q12, q21, q22, target, mode, workers):
    lib = _lib.load()
    _lib.check(lib.svb_host_apply_1q(_ptr(amps), amps.shape[0], _q(q11, q12, q21, q22), int(target)),
               "apply_single")


def apply_controlled(amps, q11, q12, q21, q22, control, target, mode, workers):
    lib = _lib.load()
    _lib.check(lib.svb_host_apply_c1q(_ptr(amps), amps.shape[0], _q(q11, q12, q21, q22),
                                      int(control), int(target)), "apply_controlled")
