"""Peer-memory transport of the multi-process engine (DistEngine(peer=True)):
2 and 4 processes on one GPU (CUDA IPC), gloo control plane, against the
oracle -- see tests/peer_ranks.py.  Covers the device-side pairwise sync
(svb_stream_signal / svb_stream_wait) and the host-barrier fallback."""
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_peer_transport_ranks_vs_oracle(cuda_ok, world):
    port = str(29600 + world)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr=127.0.0.1", f"--master-port={port}",
                        os.path.join(REPO, "tests", "peer_ranks.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert r.stdout.count(" ok") == 6, r.stdout
