"""Cold start of the runtime-specialised passes.

* jit="async" (SVB_RUN_JIT_ASYNC): the first call of a new circuit runs on
  the interpreter (a quickly planned k_fused run) while a background thread
  plans and NVRTC-compiles the specialised passes; after svb_jit_wait the
  next call runs them.  Both results match the oracle within 1e-12, and the
  post-switch result is bit-identical to the synchronous jit=True path (same
  plan, same kernels).
* the on-disk cubin cache: a second process with the same SVB_JIT_CACHE
  directory compiles nothing (every cubin is a disk hit) and gets the same
  bits.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1801_01037_b200 import _lib, device, workloads as w

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_async_jit_switches_over_and_matches(cuda_ok):
    n = 18
    circ = w.random_layer_circuit(n, 12, seed=4242)
    a0 = w.random_state_array(np.random.default_rng(5), n)
    want = oracle.run_ops(a0.copy(), w.oracle_ops(circ))
    first = device.simulate(circ, a0.copy(), fma=True, jit="async")  # interpreter, compile in background
    assert np.max(np.abs(first - want)) <= 1e-12
    _lib.jit_wait()
    launches0 = _lib.launch_count()
    second = device.simulate(circ, a0.copy(), fma=True, jit="async")  # specialised passes now
    assert np.max(np.abs(second - want)) <= 1e-12
    sync = device.simulate(circ, a0.copy(), fma=True, jit=True)
    assert np.array_equal(second, sync)
    assert _lib.launch_count() > launches0


_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r})
from paper_1801_01037_b200 import _lib, device, workloads as w
circ = w.random_layer_circuit(17, 10, seed=777)
out = device.simulate(circ, None, fma=True, jit=True)
np.save({path!r}, out)
print(*_lib.jit_counters())
"""


def test_disk_cache_second_process_compiles_nothing(cuda_ok, tmp_path):
    env = dict(os.environ, SVB_JIT_CACHE=str(tmp_path / "cache"))
    res = []
    for k in range(2):
        path = str(tmp_path / f"out{k}.npy")
        r = subprocess.run([sys.executable, "-c", _CHILD.format(repo=REPO, path=path)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        hits, comps = map(int, r.stdout.split()[-2:])
        res.append((hits, comps, np.load(path)))
    assert res[0][0] == 0 and res[0][1] > 0      # first process: compiled
    assert res[1][1] == 0 and res[1][0] == res[0][1]  # second: every cubin from disk
    assert np.array_equal(res[0][2], res[1][2])
