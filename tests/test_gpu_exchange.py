"""GPU kernels of the multi-process engine (dist.CudaCompute): own-row
exchange update (scheme b / chunked, engine.py:241-272), control packing and
packed update (regime ii, engine.py:444-447), pair update (peer-memory form)
-- each against the C oracle, bit for bit.  Plus DistEngine on one rank."""

import numpy as np
import pytest

import oracle
from paper_1801_01037_b200 import rx, standard_gate
from paper_1801_01037_b200 import workloads as w

pytestmark = pytest.mark.gpu


def _gates(rng):
    return [w.random_unitary2(rng), standard_gate("h"), standard_gate("x"), rx(0.3), standard_gate("t")]


def test_exchange_own_row_chunks(cuda_ok):
    import torch

    from paper_1801_01037_b200.dist import CudaCompute

    cc = CudaCompute()
    rng = np.random.default_rng(1)
    L = 1 << 12
    for g in _gates(rng):
        for low in (True, False):
            own = w.random_state_array(rng, 12)
            other = w.random_state_array(rng, 12)
            want = oracle.exchange_own_row(own.copy(), other.copy(), g, low)
            d_own = cc.from_numpy(own)
            for off in range(0, L, 1000):  # ragged chunks, like the pipeline's tail
                cnt = min(1000, L - off)
                d_other = cc.from_numpy(other[off:off + cnt])
                cc.exchange_update(d_own, d_other, cnt, g, low, -1, 0, own_offset=off)
            torch.cuda.synchronize()
            assert np.array_equal(cc.to_numpy(d_own), want)


def test_packed_control_exchange(cuda_ok):
    import torch

    from paper_1801_01037_b200.dist import CudaCompute

    cc = CudaCompute()
    rng = np.random.default_rng(2)
    n = 11
    L = 1 << n
    for cbit in (0, 3, n - 1):
        for g in _gates(rng):
            for low in (True, False):
                own = w.random_state_array(rng, n)
                other = w.random_state_array(rng, n)
                want = oracle.exchange_own_row(own.copy(), other.copy(), g, low, cbit=cbit)
                d_own, d_other = cc.from_numpy(own), cc.from_numpy(other)
                packed = cc.zeros(L // 2)
                cc.pack(d_other, packed, L // 2, cbit, 0)
                for off in range(0, L // 2, 300):
                    cnt = min(300, L // 2 - off)
                    cc.exchange_update(d_own, packed[off:off + cnt], cnt, g, low, cbit, off)
                torch.cuda.synchronize()
                assert np.array_equal(cc.to_numpy(d_own), want)


def test_pair_update_matches_own_row(cuda_ok):
    import ctypes

    import torch

    from paper_1801_01037_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(3)
    for cbit in (-1, 2):
        g = w.random_unitary2(rng)
        lo = w.random_state_array(rng, 10)
        hi = w.random_state_array(rng, 10)
        want_lo = oracle.exchange_own_row(lo.copy(), hi.copy(), g, True, None if cbit < 0 else cbit)
        want_hi = oracle.exchange_own_row(hi.copy(), lo.copy(), g, False, None if cbit < 0 else cbit)
        d_lo = torch.from_numpy(lo.copy()).cuda()
        d_hi = torch.from_numpy(hi.copy()).cuda()
        L = lo.shape[0]
        for b, e in ((0, L // 2), (L // 2, L)):  # the two ranks' halves
            _lib.check(lib.svb_pair_update(ctypes.c_void_p(d_lo.data_ptr()), ctypes.c_void_p(d_hi.data_ptr()),
                                           b, e, _lib.gate_array(g), cbit, None))
        torch.cuda.synchronize()
        assert np.array_equal(d_lo.cpu().numpy(), want_lo)
        assert np.array_equal(d_hi.cpu().numpy(), want_hi)


def test_dist_engine_single_rank_on_gpu(cuda_ok):
    import os
    import socket

    import torch.distributed as dist

    from paper_1801_01037_b200.dist import DistEngine

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        n = 16
        circ = w.random_layer_circuit(n, 4, seed=9)
        a = w.seeded_state(n, 4)
        eng = DistEngine(n, initial=a)
        eng.run(circ)
        got = eng.gather()
        want = oracle.run_ops(a.copy(), w.oracle_ops(circ), workers=8)
        assert np.max(np.abs(got - want)) <= 1e-12
        assert abs(eng.norm2() - 1) < 1e-12
    finally:
        dist.destroy_process_group()


def test_half_slab_swap_kernels(cuda_ok):
    # svb_pack_half / svb_unpack_half: the two halves of a global<->local
    # qubit swap (DistEngine layout mode).  Emulate two ranks on one GPU and
    # check the swapped slabs against the index permutation that exchanges
    # rank bit g and local bit l.
    import torch

    from paper_1801_01037_b200.dist import CudaCompute

    cc = CudaCompute()
    rng = np.random.default_rng(3)
    n_loc = 10
    L = 1 << n_loc
    for l in (0, 4, n_loc - 1):
        slabs = [w.random_state_array(rng, n_loc) for _ in range(2)]
        full = np.concatenate(slabs)  # rank bit = bit n_loc of the global index
        d = [cc.from_numpy(x) for x in slabs]
        bufs = [cc.zeros(L // 2) for _ in range(2)]
        for r in range(2):  # rank r sends its half with bit l != r
            cc.pack_half(d[r], bufs[r], L // 2, l, 1 - r, 0)
        for r in range(2):
            for off in range(0, L // 2, 100):  # chunked, like the pipelined exchange
                cnt = min(100, L // 2 - off)
                cc.unpack_half(d[r], bufs[1 - r][off:off + cnt], cnt, l, 1 - r, off)
        torch.cuda.synchronize()
        idx = np.arange(2 * L)
        bl, bg = (idx >> l) & 1, (idx >> n_loc) & 1
        src = idx ^ ((bl ^ bg) << l) ^ ((bl ^ bg) << n_loc)  # swap the two bits
        want = full[src]
        got = np.concatenate([cc.to_numpy(x) for x in d])
        assert np.array_equal(got, want)
