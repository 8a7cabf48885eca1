"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the host mirror of the reference API validates like the reference, and the
partition / protocol-accounting logic reproduces the reference's numbers."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import REPO, gate_from_q, golden
from paper_1801_01037_b200 import (
    SCHEME_A,
    SCHEME_B,
    Circuit,
    ExecStrategy,
    GateOp,
    PartitionPlan,
    ValidationError,
    apply_controlled,
    apply_single,
    chunked,
    comm_pairs,
    comm_partner,
    make_state,
    needs_comm,
    standard_gate,
)
from paper_1801_01037_b200 import _lib, engine, workloads
from paper_1801_01037_b200.partition import protocol_accounting


def header_symbols():
    text = open(os.path.join(REPO, "include", "svb.h")).read()
    return sorted(set(re.findall(r"\b(svb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load(require_cuda=False)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_lib.EXPORTED)
    assert lib.svb_abi_version() == 1


def test_library_validation_without_gpu():
    lib = _lib.load(require_cuda=False)
    q = _lib.gate_array(standard_gate("h"))
    assert lib.svb_apply_1q(None, 8, q, 0, None) == _lib.SVB_EINVAL
    assert b"NULL" in lib.svb_last_error()
    # non power of two, bad target, equal control/target: rejected before any launch
    buf = ctypes.create_string_buffer(16 * 64 + 16)
    p = ctypes.c_void_p((ctypes.addressof(buf) + 15) // 16 * 16)
    assert lib.svb_apply_1q(p, 6, q, 0, None) == _lib.SVB_EINVAL
    assert lib.svb_apply_1q(p, 8, q, 3, None) == _lib.SVB_EINVAL
    assert lib.svb_apply_c1q(p, 8, q, 1, 1, None) == _lib.SVB_EINVAL
    assert lib.svb_apply_c1q(p, 8, q, 3, 1, None) == _lib.SVB_EINVAL
    with pytest.raises(ValidationError):
        _lib.check(lib.svb_apply_1q(p, 8, q, 3, None))


def test_plan_passes_host_only():
    from paper_1801_01037_b200 import device

    circ = workloads.random_layer_circuit(20, 2, seed=1)
    assert device.plan_passes(20, circ, fuse=False) == len(circ.ops)
    fused = device.plan_passes(20, circ, fuse=True)
    assert 1 <= fused <= len(circ.ops)


def test_jit_sources_compile_with_nvrtc():
    # host-only: every fused pass of a circuit lowers to CUDA C that NVRTC
    # compiles for sm_100a (no device needed)
    lib = _lib.load(require_cuda=False)
    circ = workloads.random_layer_circuit(15, 2, seed=4)
    arr, nops = _lib.ops_array(circ.ops)
    out = ctypes.c_int()
    rc = lib.svb_jit_check(15, arr, nops, _lib.run_flags(fma=True), ctypes.byref(out))
    if rc == _lib.SVB_ESTATE and b"NVRTC not available" in lib.svb_last_error():
        pytest.skip("NVRTC not available")
    assert rc == 0, lib.svb_last_error()
    assert out.value >= 1


def test_outside_tile_plans_host_only(monkeypatch):
    # specialised passes leave controls / diagonal targets outside the tile
    # (tile-uniform predicates): fewer passes, and the sources still compile
    from paper_1801_01037_b200 import device

    lib = _lib.load(require_cuda=False)
    out = ctypes.c_int()
    for n, circ in ((19, workloads.qft_circuit(19)), (20, workloads.random_layer_circuit(20, 20, seed=3))):
        monkeypatch.setenv("SVB_FUSE_OUTSIDE", "0")
        inside = device.plan_passes(n, circ, jit=True)
        monkeypatch.delenv("SVB_FUSE_OUTSIDE")
        arr, nops = _lib.ops_array(circ.ops)
        rc = lib.svb_jit_check(n, arr, nops, _lib.run_flags(fma=True), ctypes.byref(out))
        if rc == _lib.SVB_ESTATE and b"NVRTC not available" in lib.svb_last_error():
            pytest.skip("NVRTC not available")
        assert rc == 0, lib.svb_last_error()
        assert device.plan_passes(n, circ, jit=True) < inside
        # strict order and the interpreter keep every qubit of an op in the tile
        assert device.plan_passes(n, circ, jit=True, strict_order=True) == \
            device.plan_passes(n, circ, jit=False, strict_order=True)


def test_kernel_wrapper_validates_like_reference():
    # kernel/__init__.py:83-97, 124-128 -- raised before any device work
    with pytest.raises(ValidationError):
        apply_single(make_state(3), standard_gate("x"), 3)
    with pytest.raises(ValidationError):
        apply_controlled(make_state(3), standard_gate("x"), 1, 1)
    with pytest.raises(ValidationError):
        apply_single(np.zeros(6, np.complex128), standard_gate("x"), 0)
    with pytest.raises(ValidationError):
        apply_single(np.zeros(8, np.complex64), standard_gate("x"), 0)
    with pytest.raises(ValidationError):
        apply_single(make_state(3), standard_gate("x"), 0, backend="python")
    with pytest.raises(ValidationError):
        ExecStrategy("warp", 2)
    with pytest.raises(ValidationError):
        ExecStrategy("sequential", 0)


def test_partition_pairs_golden():
    # test_partition.py / test_acceptance.py:123-141: n=3, k=2, t=2 -> {0,2},{1,3}
    plan = PartitionPlan(3, 2)
    assert comm_pairs(plan, 2).pairs() == [(0, 2), (1, 3)]
    for n in range(2, 9):
        for k in range(1, n):
            plan = PartitionPlan(n, k)
            for i in range(n):
                assert needs_comm(plan, i) == (i >= n - k)
                if i >= n - k:
                    for r in range(plan.p):
                        assert comm_partner(plan, r, i) == r ^ (1 << (i - (n - k)))


def test_protocol_accounting_formulas():
    # test_engine.py:121-141
    for n in range(2, 11):
        for k in range(1, min(3, n - 1) + 1):
            plan = PartitionPlan(n, k)
            L = plan.local_len
            for low in (True, False):
                assert protocol_accounting(plan, SCHEME_A, low, None) == (2, 2 * 16 * 2 ** (n - k - 1))
                assert protocol_accounting(plan, SCHEME_B, low, None) == (L, 16 * L)
                for m in (1, 2, L):
                    assert protocol_accounting(plan, chunked(m), low, None) == (
                        math.ceil(L / m), 16 * m * math.ceil(L / m))


def test_protocol_stats_match_reference_run_circuit():
    z = golden("engine.npz")
    ops = z["ops"]
    pos = 0
    for case, (n, k, scheme_id, nops) in enumerate(z["meta"]):
        rows = ops[ops[:, 0] == case]
        circ = Circuit(int(n), tuple(
            GateOp("single" if r[2] < 0 else "controlled", gate_from_q(r[3:]), int(r[1]),
                   None if r[2] < 0 else int(r[2])) for r in rows))
        scheme = (SCHEME_A, SCHEME_B, chunked(2))[int(scheme_id)]
        got = engine.protocol_stats(circ, PartitionPlan(int(n), int(k)), scheme)
        want = list(zip(z["msgs"][pos:pos + nops], z["bytes"][pos:pos + nops]))
        assert [tuple(map(int, g)) for g in got] == [tuple(map(int, w_)) for w_ in want], case
        pos += nops


def test_workload_shapes():
    assert len(workloads.qft_circuit(20).ops) == 240
    assert len(workloads.random_layer_circuit(26, 200).ops) == 7800
    c5 = workloads.random_layer_circuit(34, 2, seed=5)
    assert len(c5.ops) == 2 * (34 + 17)
    sw = workloads.sweep_ops(30, 10)
    assert len(sw.ops) == 300 and [op.target for op in sw.ops[:11]] == [0] * 10 + [1]


def test_library_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1801_01037_b200 import NativeLibraryMissing, device

    with pytest.raises(NativeLibraryMissing):
        device.simulate(workloads.qft_circuit(3))


def _run_qft_host(n, x):
    import subprocess

    exe = os.path.join(REPO, "examples", "qft_host")
    if not os.path.exists(exe):
        pytest.skip("examples/qft_host not built (run build())")
    return subprocess.run([exe, str(n), str(x)], capture_output=True, text=True, timeout=300)


def test_c_abi_example_links():
    """examples/qft_host.c (a compiled caller using only include/svb.h) builds
    and links against libsvb.so; on a host without a GPU it runs up to the
    first device call and fails loudly (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: tests/test_host.py::test_c_abi_example_on_gpu runs it")
    r = _run_qft_host(6, 3)
    assert r.returncode == 2, r.stdout + r.stderr  # the library reports the missing device


@pytest.mark.gpu
def test_c_abi_example_on_gpu(cuda_ok):
    """The same C program on the B200: QFT n=18 of |12345> through
    svb_host_run_ops, every amplitude within 1e-12 of the closed form."""
    r = _run_qft_host(18, 12345)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max|err|" in r.stdout
