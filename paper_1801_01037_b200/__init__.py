"""B200-native state-vector gate engine (drop-in for svsim's apply-gate path).

Hot path: 1-qubit and controlled 2x2 unitaries on a 2^n complex128 vector,
partitioned over 2^k ranks with a partner exchange for rank-bit qubits
(BASELINE.json north_star).  Compute is hand-written sm_100a
CUDA in libsvb.so behind a C ABI (include/svb.h); PyTorch only owns device
buffers and streams.  Names mirror the reference package ``svsim``
(pkg/src/svsim/__init__.py:93-161) for the parts on this path.
"""

from .core import (
    BYTES_PER_AMPLITUDE,
    MAX_QUBITS,
    NORM_TOL,
    Circuit,
    Gate2x2,
    GateOp,
    StateVector,
    is_unitary,
    make_state,
    norm2,
    phase,
    rx,
    ry,
    rz,
    standard_gate,
)
from .errors import (
    CapacityError,
    ContractViolation,
    NativeLibraryMissing,
    ParseError,
    SvsimError,
    ValidationError,
)
from .kernel import (
    BACKEND,
    SEQUENTIAL,
    ExecStrategy,
    apply_controlled,
    apply_single,
    available_backends,
    update_pair,
)
from .partition import (
    SCHEME_A,
    SCHEME_B,
    CommScheme,
    PartitionPlan,
    RankMatching,
    chunked,
    comm_pairs,
    comm_partner,
    needs_comm,
)

__version__ = "0.1.0"

_LAZY = {
    "DeviceState": "device", "simulate": "device", "run_ops": "device", "probs": "device",
    "DistState": "engine", "GateStats": "engine", "dist_init": "engine", "gather": "engine",
    "dist_apply_local": "engine", "dist_apply_scheme_a": "engine", "dist_apply_scheme_b": "engine",
    "dist_apply_chunked": "engine", "dist_apply_controlled": "engine", "run_circuit": "engine",
    "time_ratio": "engine", "dist_norm2": "engine", "PeerTransport": "engine", "InMemoryTransport": "engine",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod = importlib.import_module(f".{_LAZY[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
