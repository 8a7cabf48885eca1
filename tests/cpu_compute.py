"""Checker-backed compute for CPU-only multi-process tests of dist.DistEngine.

TEST INFRASTRUCTURE: implements the compute interface of
paper_1801_01037_b200.dist.CudaCompute on CPU torch tensors with the C
oracle (oracle/svsim_oracle.c), so the multi-rank orchestration -- partner
selection, chunk pipelining over torch.distributed (gloo), control packing,
regime dispatch, diagonal elision -- runs here without a GPU.  The product
engine never constructs this; it is injected by tests only.
"""

import numpy as np
import torch

import oracle


def _insert_one(p: np.ndarray, cbit: int) -> np.ndarray:
    low = p & ((1 << cbit) - 1)
    return ((p >> cbit) << (cbit + 1)) | (1 << cbit) | low


def _insert(p: np.ndarray, bit: int, value: int) -> np.ndarray:
    low = p & ((1 << bit) - 1)
    return ((p >> bit) << (bit + 1)) | (value << bit) | low


class CpuCompute:
    def zeros(self, count):
        return torch.zeros(count, dtype=torch.complex128)

    def flag_words(self, count):  # peer-transport sync words (never signalled on CPU)
        return torch.zeros(count, dtype=torch.int32)

    def from_numpy(self, arr):
        return torch.from_numpy(np.ascontiguousarray(arr).copy())

    def to_numpy(self, t):
        return t.numpy().copy()

    def run_ops(self, slab, ops, fuse=True, strict=False, fma=False, jit=False):
        a = slab.numpy()
        oracle.run_ops(a, [(op.gate, op.target, op.control) for op in ops])

    def pack_half(self, src, dst, count, bit, value, offset):
        idx = _insert(np.arange(offset, offset + count, dtype=np.int64), bit, value)
        dst.numpy()[:count] = src.numpy()[idx]

    def unpack_half(self, dst, src, count, bit, value, offset):
        idx = _insert(np.arange(offset, offset + count, dtype=np.int64), bit, value)
        dst.numpy()[idx] = src.numpy()[:count]

    def pack(self, src, dst, count, cbit, offset):
        idx = _insert_one(np.arange(offset, offset + count, dtype=np.int64), cbit)
        dst.numpy()[:count] = src.numpy()[idx]

    def exchange_update(self, own, other, count, gate, own_is_low, cbit, offset, own_offset=0):
        o = other.numpy()[:count].copy()
        if cbit < 0:
            view = own.numpy()[own_offset:own_offset + count]
            tmp = view.copy()
            oracle.exchange_own_row(tmp, o, gate, own_is_low)
            view[:] = tmp
        else:
            idx = _insert_one(np.arange(offset, offset + count, dtype=np.int64), cbit)
            tmp = own.numpy()[idx].copy()
            oracle.exchange_own_row(tmp, o, gate, own_is_low)
            own.numpy()[idx] = tmp

    def norm2(self, slab):
        return oracle.norm2(slab.numpy())

    def synchronize(self):
        pass
