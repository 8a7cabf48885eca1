"""Rank partitioning of the amplitude index space (pkg/src/svsim/partition.py).

2^k ranks split 2^n amplitudes into contiguous slabs: rank r owns global
indices [r * 2^(n-k), (r+1) * 2^(n-k)) (partition.py:3-6, 52-56).  A gate on
qubit i is rank-local iff i < n-k (partition.py:119-123); otherwise rank r
pairs with r ^ 2^(i-(n-k)) (partition.py:126-137), a perfect matching
(partition.py:140-159).  One rank = one GPU (or one slab of an emulated
multi-rank run on a single GPU).

Also here: the reference's exchange protocols (CommScheme, partition.py:59-96)
and their exact per-rank message/byte formulas (engine.py:8-18, 206-272),
so GateStats keeps the reference's accounting semantics.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .core import BYTES_PER_AMPLITUDE
from .errors import ContractViolation, ValidationError


@dataclass(frozen=True)
class PartitionPlan:
    """n qubits over 2**k ranks (partition.py:26-56)."""

    n: int
    k: int

    def __post_init__(self):
        if self.n < 1:
            raise ValidationError(f"need at least one qubit, got n={self.n}")
        if not (0 <= self.k <= self.n - 1):
            raise ValidationError(
                f"k must lie in [0, n-1] so each rank holds at least a pair, got k={self.k} for n={self.n}")

    @property
    def p(self) -> int:
        return 1 << self.k

    @property
    def local_len(self) -> int:
        return 1 << (self.n - self.k)

    def rank_of(self, gindex: int) -> int:
        return gindex >> (self.n - self.k)

    def first_index(self, rank: int) -> int:
        return rank << (self.n - self.k)


@dataclass(frozen=True)
class CommScheme:
    """Exchange protocol selector (partition.py:59-88)."""

    kind: str
    m: int | None = None

    def __post_init__(self):
        if self.kind not in ("a", "b", "chunked"):
            raise ValidationError(f"unknown scheme kind {self.kind!r}")
        if self.kind == "chunked":
            if not isinstance(self.m, int) or self.m < 1:
                raise ValidationError(f"chunk size must be an int >= 1, got {self.m!r}")
        elif self.m is not None:
            raise ValidationError(f"scheme {self.kind!r} takes no chunk size")

    def buffer_amps(self, plan: PartitionPlan) -> int:
        if plan.k == 0:
            return 0
        if self.kind == "a":
            return plan.local_len // 2
        if self.kind == "b":
            return 1
        if self.m > plan.local_len:
            raise ValidationError(f"chunk size {self.m} exceeds slab length {plan.local_len}")
        return self.m


SCHEME_A = CommScheme("a")
SCHEME_B = CommScheme("b")


def chunked(m: int) -> CommScheme:
    return CommScheme("chunked", m)


@dataclass(frozen=True)
class RankMatching:
    """partition.py:99-116."""

    qubit: int
    partner_of: tuple[int, ...]

    def __post_init__(self):
        po = self.partner_of
        for r, q in enumerate(po):
            if q == r or not (0 <= q < len(po)) or po[q] != r:
                raise ValidationError(f"not a fixed-point-free involution at rank {r}: partner {q}")

    def pairs(self) -> list[tuple[int, int]]:
        return [(r, q) for r, q in enumerate(self.partner_of) if r < q]


def needs_comm(plan: PartitionPlan, i: int) -> bool:
    if not (0 <= i < plan.n):
        raise ValidationError(f"qubit {i} out of range for n={plan.n}")
    return i >= plan.n - plan.k


def comm_partner(plan: PartitionPlan, rank: int, i: int) -> int:
    if not (0 <= rank < plan.p):
        raise ValidationError(f"rank {rank} out of range for p={plan.p}")
    if not needs_comm(plan, i):
        raise ContractViolation(f"qubit {i} is rank-local for n={plan.n}, k={plan.k}")
    return (plan.first_index(rank) ^ (1 << i)) >> (plan.n - plan.k)


def comm_pairs(plan: PartitionPlan, i: int) -> RankMatching:
    if not needs_comm(plan, i):
        raise ContractViolation(f"qubit {i} is rank-local for n={plan.n}, k={plan.k}")
    partner_of = [-1] * plan.p
    for r in range(plan.p):
        if partner_of[r] < 0:
            q = comm_partner(plan, r, i)
            partner_of[r], partner_of[q] = q, r
    return RankMatching(i, tuple(partner_of))


def _count_bit_set(lo: int, hi: int, cbit: int | None) -> int:
    """#indices j in [lo, hi) with bit cbit set (all of them when cbit is None)."""
    if cbit is None:
        return hi - lo

    def f(x: int) -> int:
        period = 1 << (cbit + 1)
        return (x // period) * (1 << cbit) + max(0, (x % period) - (1 << cbit))

    return f(hi) - f(lo)


def protocol_accounting(plan: PartitionPlan, scheme: CommScheme, low: bool,
                        cbit: int | None) -> tuple[int, int]:
    """(messages, bytes) one rank sends for one exchange under the reference
    protocol (engine.py:206-272)."""
    L = plan.local_len
    if scheme.kind == "a":
        half = L >> 1
        ship = _count_bit_set(half, L, cbit) if low else _count_bit_set(0, half, cbit)
        work = _count_bit_set(0, half, cbit) if low else _count_bit_set(half, L, cbit)
        msgs = (1 if ship else 0) + (1 if work else 0)
        return msgs, BYTES_PER_AMPLITUDE * (ship + work)
    count = _count_bit_set(0, L, cbit)
    if scheme.kind == "b":
        return count, BYTES_PER_AMPLITUDE * count
    chunks = math.ceil(count / scheme.m)
    return chunks, BYTES_PER_AMPLITUDE * scheme.m * chunks
