"""Shared test setup.

Marker ``gpu``: needs a B200 (run with ``-m gpu`` on the GPU box).  Tests
without it run on CPU in the build container.  ``oracle/`` is importable
here as the checker; the product package never imports it.
"""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def split_cases(meta_n, flat):
    """Split concatenated per-case amplitude arrays by 2**n lengths."""
    out, pos = [], 0
    for n in meta_n:
        ln = 1 << int(n)
        out.append(flat[pos:pos + ln])
        pos += ln
    return out


def gate_from_q(q):
    from paper_1801_01037_b200.core import Gate2x2

    return Gate2x2(complex(q[0], q[1]), complex(q[2], q[3]), complex(q[4], q[5]),
                   complex(q[6], q[7]))


def circuit_from_rows(n, rows):
    """Rebuild a circuit from golden op rows [target, control|-1, q0..q7]."""
    from paper_1801_01037_b200.core import Circuit, GateOp

    ops = []
    for r in rows:
        t, c = int(r[0]), int(r[1])
        g = gate_from_q(r[2:])
        ops.append(GateOp("single", g, t) if c < 0 else GateOp("controlled", g, t, c))
    return Circuit(int(n), tuple(ops))


@pytest.fixture(scope="session")
def cuda_ok():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
