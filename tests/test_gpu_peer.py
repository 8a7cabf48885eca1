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


@pytest.mark.gpu
def test_multi_gpu_bench_path_smoke(cuda_ok):
    """bench.py --gpus 2 (configs[3] QFT path, reference-faithful mode,
    configs[4] path) with both ranks on one GPU over a gloo control plane:
    the line prints and its known-answer / round-trip checks pass."""
    import json

    env = dict(os.environ, SVB_DIST_BACKEND="gloo", SVB_BENCH_QFT_N="22", SVB_BENCH_CFG4="1",
               SVB_BENCH_CFG4_N="22")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29611", os.path.join(REPO, "bench.py"),
                        "--gpus", "2", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["check"]["pass"], line["check"]
    assert line["nvlink"]["global_ops"] > 0 and line["reference_faithful"]["exchanges_per_step"] > 0
    assert abs(line["configs4"]["norm_after"] - 1.0) < 1e-12
    # the timed regions run on cached plans: settle runs after the warm-ups
    # (layout mode), configs[4] from |0...0> after an untimed run of the same kind
    assert 1 <= line["settle_runs"] <= 8 and "identity layout" in line["configs4"]["step"]
