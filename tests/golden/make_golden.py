"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies the read-only reference package to a scratch dir, builds its
compiled Cython kernel there with the reference's own setup.py (system gcc,
SURVEY 7 step 0), imports ``svsim`` and records inputs/outputs of the
reference's public API:

* kernel_single.npz / kernel_controlled.npz: the 200-case random loops of
  pkg/tests/test_kernel.py:72-82 and 107-117 (seeds 21, 22), outputs of the
  compiled backend (``apply_single`` / ``apply_controlled``).
* engine.npz: ``run_circuit`` on random circuits (pkg/tests/conftest.py:32-43)
  over PartitionPlan(n, k), schemes a / b / chunked(2); gathered amplitudes
  plus per-gate GateStats messages/bytes (engine.py:457-512).
* qft.npz: config 1 -- QFT n=20 on the seeded Gaussian state, compiled
  backend, sequential strategy (the paper's mode); full output at n=12, and
  at n=20 a sha256 of the canonicalised bytes plus 4096 sampled amplitudes.
* layers.npz: config-2 style random layer circuit at n=12, 20 layers, from
  |0...0>, compiled backend.

Nothing here runs on the GPU box; the .npz files are committed.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
SCRATCH = "/tmp/svsim_golden_build"


def build_reference():
    if os.path.exists(SCRATCH):
        shutil.rmtree(SCRATCH)
    shutil.copytree(REF, SCRATCH)
    env = dict(os.environ, CC="/usr/bin/gcc", LDSHARED="/usr/bin/gcc -shared")
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                   env=env, check=True, capture_output=True)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    sys.path.insert(0, os.path.join(SCRATCH, "tests"))
    import svsim

    assert svsim.available_backends() == ("python", "compiled"), svsim.available_backends()
    return svsim


def canon_sha(a: np.ndarray) -> str:
    """sha256 of the amplitude bytes with -0.0 folded to +0.0 (x + 0.0)."""
    v = np.ascontiguousarray(a, dtype=np.complex128).view(np.float64) + 0.0
    return hashlib.sha256(v.tobytes()).hexdigest()


def gq(g) -> np.ndarray:
    return np.array([v for z in (g.q11, g.q12, g.q21, g.q22)
                     for v in (complex(z).real, complex(z).imag)])


def kernel_cases(svsim, conftest, seed: int, controlled: bool):
    rng = np.random.default_rng(seed)
    meta, gates, ins, outs = [], [], [], []
    for _ in range(200):
        if controlled:
            n = int(rng.integers(2, 9))
            c, t = (int(v) for v in rng.choice(n, size=2, replace=False))
        else:
            n = int(rng.integers(1, 9))
            t = int(rng.integers(n))
            c = -1
        g = conftest.random_unitary2(rng)
        a = conftest.random_state_array(rng, n)
        s = svsim.StateVector(n, a.copy())
        if controlled:
            svsim.apply_controlled(s, g, c, t, backend="compiled")
        else:
            svsim.apply_single(s, g, t, backend="compiled")
        meta.append((n, c, t))
        gates.append(gq(g))
        ins.append(a)
        outs.append(s.amps.copy())
    return dict(meta=np.array(meta), gates=np.array(gates), inp=np.concatenate(ins),
                out=np.concatenate(outs))


def engine_cases(svsim, conftest):
    rng = np.random.default_rng(4242)
    cases = {"meta": [], "gates": [], "ops": [], "out": [], "msgs": [], "bytes": []}
    op_rows = []
    for case in range(60):
        n = int(rng.integers(2, 11))
        k = int(rng.integers(0, min(3, n - 1) + 1))
        scheme_id = int(rng.integers(3))
        scheme = (svsim.SCHEME_A, svsim.SCHEME_B, svsim.chunked(2))[scheme_id]
        if scheme_id == 1 and n - k > 8:
            scheme_id, scheme = 2, svsim.chunked(2)
        circ = conftest.random_circuit(rng, n, 12)
        ds, stats = svsim.run_circuit(circ, svsim.PartitionPlan(n, k), scheme)
        out = svsim.gather(ds).amps
        for op in circ.ops:
            op_rows.append([case, op.target, -1 if op.control is None else op.control, *gq(op.gate)])
        cases["meta"].append((n, k, scheme_id, len(circ.ops)))
        cases["out"].append(out)
        cases["msgs"] += [st.messages_sent_per_rank for st in stats]
        cases["bytes"] += [st.bytes_sent_per_rank for st in stats]
    return dict(meta=np.array(cases["meta"]), ops=np.array(op_rows),
                out=np.concatenate(cases["out"]), msgs=np.array(cases["msgs"]),
                bytes=np.array(cases["bytes"]))


def op_rows(circ) -> np.ndarray:
    """[target, control (-1), 8 gate doubles] per op: the exact gate bits, so
    tests never depend on the host's libm/LAPACK rounding when rebuilding."""
    return np.array([[op.target, -1 if op.control is None else op.control, *gq(op.gate)]
                     for op in circ.ops])


def run_ref(svsim, amps, circ, strat):
    s = svsim.StateVector(circ.n, amps, validate=False)
    for op in circ.ops:
        g = svsim.Gate2x2(op.gate.q11, op.gate.q12, op.gate.q21, op.gate.q22)
        if op.control is None:
            svsim.apply_single(s, g, op.target, strat=strat, backend="compiled")
        else:
            svsim.apply_controlled(s, g, op.control, op.target, strat=strat, backend="compiled")
    return s.amps


def main():
    svsim = build_reference()
    import conftest  # the reference's own test helpers

    sys.path.insert(0, REPO)
    from paper_1801_01037_b200 import workloads as w

    np.savez_compressed(os.path.join(HERE, "kernel_single.npz"),
                        **kernel_cases(svsim, conftest, 21, False))
    np.savez_compressed(os.path.join(HERE, "kernel_controlled.npz"),
                        **kernel_cases(svsim, conftest, 22, True))
    np.savez_compressed(os.path.join(HERE, "engine.npz"), **engine_cases(svsim, conftest))

    seq = svsim.ExecStrategy("sequential", 1)
    q = {}
    for n in (12, 20):
        # seeded_state: host-independent normalisation (fsum, no BLAS)
        a = w.seeded_state(n, w.SEED_STATE)
        circ = w.qft_circuit(n)
        q[f"ops{n}"] = op_rows(circ)
        out = run_ref(svsim, a.copy(), circ, seq)
        q[f"sha{n}"] = np.array(canon_sha(out))
        q[f"in_sha{n}"] = np.array(canon_sha(a))
        q[f"norm{n}"] = np.array(float(np.vdot(out, out).real))
        idx = np.random.default_rng(99).choice(1 << n, size=min(4096, 1 << n), replace=False)
        q[f"idx{n}"] = idx
        q[f"amp{n}"] = out[idx]
        q[f"prob{n}"] = np.abs(out[idx]) ** 2
        if n == 12:
            q["out12"] = out
    np.savez_compressed(os.path.join(HERE, "qft.npz"), **q)

    circ = w.random_layer_circuit(12, 20, seed=w.SEED_CFG2)
    a = np.zeros(1 << 12, np.complex128)
    a[0] = 1
    out = run_ref(svsim, a, circ, svsim.ExecStrategy("parallel_collapsed", 4))
    np.savez_compressed(os.path.join(HERE, "layers.npz"), out=out, sha=np.array(canon_sha(out)),
                        ops=op_rows(circ),
                        n=np.array(12), layers=np.array(20), seed=np.array(w.SEED_CFG2))
    import json

    texts = [
        "qubits 3\nh 0\ncx 0 1\nz 2  # trailing\n\n# comment\nu 1 0 0 1 0 1 0 0 0\n",
        "qubits 2\ncu 1 0 1 0 0 0 0 0 0 1\ncy 0 1\n",
        "qubits 2\nq 0\n",
        "h 0\n",
        "qubits 2\nx 2\n",
        "qubits 2\ncx 1 1\n",
        "qubits 2\nu 0 1 0 1 0 0 0 1 0\n",
        "qubits 2\nu 0 1 0 0 0 0 0 1\n",
        "qubits 0\n",
        "qubits 2\nx one\n",
        "",
    ]
    cases = []
    for txt in texts:
        try:
            c = svsim.parse_circuit(txt)
            cases.append({"text": txt, "n": c.n, "ops": op_rows(c).tolist()})
        except svsim.ParseError as exc:
            cases.append({"text": txt, "error_line": exc.line})
    fmt = []
    rng = np.random.default_rng(11)
    for circ in (w.qft_circuit(5), conftest.random_circuit(rng, 4, 12)):
        rc = svsim.Circuit(circ.n, tuple(svsim.GateOp(op.kind, svsim.Gate2x2(op.gate.q11, op.gate.q12,
                                                                             op.gate.q21, op.gate.q22),
                                                      op.target, op.control) for op in circ.ops))
        fmt.append({"ops": op_rows(rc).tolist(), "n": rc.n, "text": svsim.format_circuit(rc)})
    with open(os.path.join(HERE, "circuit_io.json"), "w") as fh:
        json.dump({"parse": cases, "format": fmt}, fh, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
