"""CPU oracle for the gate-application hot path.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product
package `paper_1801_01037_b200`, which fails loudly without its CUDA library.

Three checkers live here:

* ``liboracle.so`` (oracle/svsim_oracle.c): a plain-C restatement of the
  reference's pair update, controlled sweep, own-row exchange and norm
  (cites in that file).  Bit-identical to the reference's compiled kernel.
* ``oracle/_ref/_stride_cy*.so``: the reference's OWN Cython kernel
  (pkg/src/svsim/kernel/_stride_cy.pyx) compiled from /root/reference by
  oracle/build_ref.sh.  Present wherever build() ran with the reference
  mounted; travels to the GPU box as a built file.
* dense embedding + row matvec for n <= 12, restating the reference's
  independent oracle (pkg/src/svsim/oracle.py:83-137).

Parity pinning: tests/test_oracle_golden.py checks all of these against the
golden vectors in tests/golden/, which tests/golden/make_golden.py produced by
importing the reference package itself.
"""

from __future__ import annotations

import ctypes
import glob
import importlib.machinery
import importlib.util
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_dptr = ctypes.POINTER(ctypes.c_double)


def _build_if_missing() -> str:
    path = os.path.join(HERE, "liboracle.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return path


def lib():
    """ctypes handle on liboracle.so (built on demand with gcc)."""
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(_build_if_missing())
        i64, c_int = ctypes.c_int64, ctypes.c_int
        L.or_apply_single.argtypes = [_dptr, i64, _dptr, c_int, c_int]
        L.or_apply_controlled.argtypes = [_dptr, i64, _dptr, c_int, c_int, c_int]
        L.or_apply_single_reps.argtypes = [_dptr, i64, _dptr, c_int, c_int, c_int]
        L.or_exchange_own_row.argtypes = [_dptr, _dptr, i64, _dptr, c_int, c_int]
        L.or_norm2.argtypes = [_dptr, i64]
        L.or_norm2.restype = ctypes.c_double
        L.or_probs.argtypes = [_dptr, i64, _dptr]
        L.or_max_threads.restype = c_int
        _LIB = L
    return _LIB


def ref_module():
    """The reference's own compiled kernel module, or None if not built."""
    global _REF
    if _REF is None:
        hits = glob.glob(os.path.join(HERE, "_ref", "_stride_cy*.so"))
        if not hits:
            return None
        loader = importlib.machinery.ExtensionFileLoader("_stride_cy", hits[0])
        spec = importlib.util.spec_from_file_location("_stride_cy", hits[0], loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _REF = mod
    return _REF


def _p(a: np.ndarray):
    assert a.dtype in (np.complex128, np.float64) and a.flags.c_contiguous
    return a.ctypes.data_as(_dptr)


def gate_q(g) -> np.ndarray:
    """Gate (anything with q11..q22, or a 2x2 matrix) -> 8 doubles."""
    if hasattr(g, "q11"):
        ent = (g.q11, g.q12, g.q21, g.q22)
    else:
        m = np.asarray(g, dtype=np.complex128)
        ent = (m[0, 0], m[0, 1], m[1, 0], m[1, 1])
    return np.array([v for z in ent for v in (complex(z).real, complex(z).imag)])


def apply_single(amps: np.ndarray, g, t: int, workers: int = 1) -> np.ndarray:
    q = gate_q(g)
    lib().or_apply_single(_p(amps), amps.shape[0], _p(q), int(t), int(workers))
    return amps


def apply_single_reps(amps: np.ndarray, g, t: int, reps: int, workers: int = 1) -> np.ndarray:
    """`reps` applications of g on t; bit-identical to calling apply_single
    `reps` times (each pair's update depends on that pair only)."""
    q = gate_q(g)
    lib().or_apply_single_reps(_p(amps), amps.shape[0], _p(q), int(t), int(reps), int(workers))
    return amps


def apply_controlled(amps: np.ndarray, g, c: int, t: int, workers: int = 1) -> np.ndarray:
    q = gate_q(g)
    lib().or_apply_controlled(_p(amps), amps.shape[0], _p(q), int(c), int(t), int(workers))
    return amps


def exchange_own_row(own: np.ndarray, other: np.ndarray, g, own_is_low: bool,
                     cbit: int | None = None) -> np.ndarray:
    q = gate_q(g)
    lib().or_exchange_own_row(_p(own), _p(other), own.shape[0], _p(q), int(own_is_low),
                              -1 if cbit is None else int(cbit))
    return own


def norm2(amps: np.ndarray) -> float:
    return float(lib().or_norm2(_p(amps), amps.shape[0]))


def probs(amps: np.ndarray) -> np.ndarray:
    out = np.empty(amps.shape[0], dtype=np.float64)
    lib().or_probs(_p(amps), amps.shape[0], _p(out))
    return out


def run_ops(amps: np.ndarray, ops, workers: int = 1) -> np.ndarray:
    """Apply a sequence of (gate, target, control|None) in order, in place."""
    for g, t, c in ops:
        if c is None:
            apply_single(amps, g, t, workers)
        else:
            apply_controlled(amps, g, c, t, workers)
    return amps


def run_partitioned(slabs: list[np.ndarray], n: int, ops) -> list[np.ndarray]:
    """Reference distributed semantics on 2^k host slabs (engine.py:457-512,
    scheme b own-row exchange, controlled regimes engine.py:415-450)."""
    p = len(slabs)
    k = p.bit_length() - 1
    boundary = n - k
    for g, t, c in ops:
        if c is not None and c >= boundary:
            parts = [r for r in range(p) if (r >> (c - boundary)) & 1]
        else:
            parts = list(range(p))
        if t < boundary:
            for r in parts:
                if c is None or c >= boundary:
                    apply_single(slabs[r], g, t)
                else:
                    apply_controlled(slabs[r], g, c, t)
            continue
        cbit = c if (c is not None and c < boundary) else None
        snap = {r: slabs[r].copy() for r in parts}
        for r in parts:
            partner = r ^ (1 << (t - boundary))
            exchange_own_row(slabs[r], snap[partner], g, r < partner, cbit)
    return slabs


# ---------------------------------------------------------------------------
# dense oracle (restates pkg/src/svsim/oracle.py:83-137), n <= 12


def embed_single(m: np.ndarray, i: int, n: int) -> np.ndarray:
    lower = np.eye(1 << i, dtype=np.complex128)
    upper = np.eye(1 << (n - 1 - i), dtype=np.complex128)
    return np.kron(upper, np.kron(np.asarray(m, np.complex128), lower))


def embed_controlled(m: np.ndarray, c: int, t: int, n: int) -> np.ndarray:
    m = np.asarray(m, np.complex128)
    dim = 1 << n
    e = np.eye(dim, dtype=np.complex128)
    j = np.arange(dim)
    base = j[((j >> t) & 1 == 0) & ((j >> c) & 1 == 1)]
    mate = base | (1 << t)
    e[base, base] = m[0, 0]
    e[base, mate] = m[0, 1]
    e[mate, base] = m[1, 0]
    e[mate, mate] = m[1, 1]
    return e


def dense_run(amps: np.ndarray, n: int, ops) -> np.ndarray:
    assert n <= 12
    s = np.array(amps, dtype=np.complex128)
    for g, t, c in ops:
        m = np.array([[g.q11, g.q12], [g.q21, g.q22]]) if hasattr(g, "q11") else g
        u = embed_single(m, t, n) if c is None else embed_controlled(m, c, t, n)
        s = u @ s
    return s


# ---------------------------------------------------------------------------
# QFT known answers; LSB-convention QFT as built by
# paper_1801_01037_b200.workloads.qft_ops: out = (sqrt(N) * ifft(a[br]))[br]


def bit_reverse_perm(n: int) -> np.ndarray:
    idx = np.arange(1 << n, dtype=np.int64)
    out = np.zeros_like(idx)
    for b in range(n):
        out |= ((idx >> b) & 1) << (n - 1 - b)
    return out


def qft_reference(amps: np.ndarray, n: int) -> np.ndarray:
    br = bit_reverse_perm(n)
    return (np.sqrt(1 << n) * np.fft.ifft(amps[br]))[br]


def bit_reverse_int(x: int, n: int) -> int:
    return int(format(x, f"0{n}b")[::-1], 2)


def qft_basis_amplitude(x: int, y: int, n: int) -> complex:
    """<y| QFT_lsb |x> = exp(2 pi i br(x) br(y) / N) / sqrt(N), phase reduced
    exactly in integers (no overflow at n=34)."""
    N = 1 << n
    ph = (bit_reverse_int(x, n) * bit_reverse_int(y, n)) % N
    return complex(np.exp(2j * np.pi * ph / N) / np.sqrt(N))
