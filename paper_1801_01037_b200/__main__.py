"""Command line on the B200 engine, mirroring the reference CLI's `run`,
`verify` and `bench` subcommands (pkg/src/svsim/cli.py:127-169, 206-247).

    python -m paper_1801_01037_b200 run circ.txt [--ranks P] [--scheme b]
        [--layout auto|none] [--out FILE] [--fused]
    python -m paper_1801_01037_b200 verify circ.txt [--ranks P] [--scheme b] [--fused]
    python -m paper_1801_01037_b200 bench --qubits N [--ranks P] [--gate h] [--repeat R]

`verify` runs the circuit on the engine and on the dense verifier (the GPU
matvec of dense.py, capped at 12 qubits like oracle.py:22), prints
`max deviation = X` and exits 0 iff X <= 1e-10 (cli.py:159-169, VERIFY_TOL
cli.py:47), else 1.

`run` writes `index,re,im` lines (repr floats, cli.py:111-120) and, unless
--fused, `<out>.stats.csv` with the reference's GateStats columns
(cli.py:42-45).  Exit codes: 2 parse/validation, 3 capacity (cli.py:363-376).
"""

from __future__ import annotations

import argparse
import statistics
import sys

import numpy as np

from .errors import CapacityError, ParseError, SvsimError, ValidationError

VERIFY_TOL = 1e-10  # cli.py:47
STATS_HEADER = "gate_index,qubit,control,comm_required,messages_per_rank,bytes_per_rank,wall_time_s"


def _k(ranks: int) -> int:
    if ranks < 1 or ranks & (ranks - 1):
        raise ValidationError(f"rank count must be a power of two, got {ranks}")
    return ranks.bit_length() - 1


def _scheme(text: str):
    from .partition import SCHEME_A, SCHEME_B, chunked

    t = text.strip().lower()
    if t == "a":
        return SCHEME_A
    if t == "b":
        return SCHEME_B
    if t.startswith("chunked:"):
        return chunked(int(t.split(":", 1)[1]))
    raise ValidationError(f"unknown scheme {text!r} (expected a, b, or chunked:m)")


def _stats_csv(stats) -> str:
    out = [STATS_HEADER]
    for i, st in enumerate(stats):
        ctl = "" if st.control is None else str(st.control)
        out.append(f"{i},{st.qubit},{ctl},{'true' if st.comm_required else 'false'},"
                   f"{st.messages_sent_per_rank},{st.bytes_sent_per_rank},{repr(float(st.wall_time))}")
    return "\n".join(out) + "\n"


def cmd_run(args) -> int:
    from . import device, engine
    from .circuit_io import parse_circuit_file
    from .layout import gate_histogram, optimize_layout, permute_state
    from .partition import PartitionPlan

    circuit = parse_circuit_file(args.circuit)
    if args.fused:
        amps = device.simulate(circuit)
        stats = None
    else:
        plan = PartitionPlan(circuit.n, _k(args.ranks))
        perm = optimize_layout(gate_histogram(circuit), plan.k) if args.layout == "auto" else None
        ds, stats = engine.run_circuit(circuit, plan, _scheme(args.scheme), perm=perm)
        st = engine.gather(ds)
        ds.close()
        amps = (permute_state(st, perm.inverse()) if perm is not None else st).amps
    lines = [f"{i},{repr(float(z.real))},{repr(float(z.imag))}" for i, z in enumerate(amps)]
    text = "\n".join(lines) + "\n"
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
        if stats is not None:
            with open(args.out + ".stats.csv", "w") as fh:
                fh.write(_stats_csv(stats))
    else:
        sys.stdout.write(text)
    return 0


def cmd_verify(args) -> int:
    from . import dense, device, engine
    from .circuit_io import parse_circuit_file
    from .partition import PartitionPlan

    circuit = parse_circuit_file(args.circuit)
    plan = PartitionPlan(circuit.n, _k(args.ranks))
    scheme = _scheme(args.scheme)
    expected = dense.oracle_run(circuit)  # enforces the dense verifier's qubit cap
    if args.fused:
        got = device.simulate(circuit, fuse=True)
    else:
        ds, _ = engine.run_circuit(circuit, plan, scheme)
        got = engine.gather(ds).amps
        ds.close()
    dev = float(np.max(np.abs(got - expected.amps)))
    print(f"max deviation = {dev:.3e}")
    return 0 if dev <= VERIFY_TOL else 1


def cmd_bench(args) -> int:
    """Per-qubit timing of repeated single-qubit gates through the engine, in
    the reference's output format (cli.py:206-247): header, `c = ...`, one
    line per qubit (median wall time, messages, bytes), `T = ...`, then the
    GateStats CSV."""
    from . import engine
    from .core import Circuit, GateOp, standard_gate
    from .partition import PartitionPlan

    plan = PartitionPlan(args.qubits, _k(args.ranks))
    scheme = _scheme(args.scheme)
    g = standard_gate(args.gate)
    if args.repeat < 1:
        raise ValidationError("--repeat must be >= 1")
    print(f"qubits {plan.n}  ranks {plan.p} (k = {plan.k})  scheme {args.scheme.lower()}  "
          f"gate {args.gate.lower()}  repeat {args.repeat}")
    print("c = no communication" if plan.k == 0 else f"c = {(plan.n - plan.k) / plan.k:.2f}")
    ops = tuple(GateOp("single", g, q) for q in range(plan.n) for _ in range(args.repeat))
    ds, stats = engine.run_circuit(Circuit(plan.n, ops), plan, scheme)
    ds.close()
    local, comm = [], []
    for q in range(plan.n):
        chunk = stats[q * args.repeat:(q + 1) * args.repeat]
        times = [st.wall_time for st in chunk]
        (comm if chunk[0].comm_required else local).extend(times)
        print(f"qubit {q}: median {statistics.median(times):.3e} s  "
              f"messages {chunk[0].messages_sent_per_rank}  bytes {chunk[0].bytes_sent_per_rank}")
    if comm and local:
        print(f"T = {statistics.median(comm) / statistics.median(local):.6g}")
    else:
        print("T = n/a")
    print()
    sys.stdout.write(_stats_csv(stats))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1801_01037_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("circuit")
    r.add_argument("--ranks", type=int, default=1)
    r.add_argument("--scheme", default="b")
    r.add_argument("--layout", choices=("auto", "none"), default="none")
    r.add_argument("--out")
    r.add_argument("--fused", action="store_true", help="single rank, fused passes, no per-gate stats")
    v = sub.add_parser("verify")
    v.add_argument("circuit")
    v.add_argument("--ranks", type=int, default=1)
    v.add_argument("--scheme", default="b")
    v.add_argument("--fused", action="store_true", help="check the fused single-rank path instead")
    b = sub.add_parser("bench")
    b.add_argument("--qubits", type=int, required=True)
    b.add_argument("--ranks", type=int, default=1)
    b.add_argument("--scheme", default="b")
    b.add_argument("--gate", default="h")
    b.add_argument("--repeat", type=int, default=3)
    args = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "verify": cmd_verify, "bench": cmd_bench}[args.cmd](args)
    except (ParseError, ValidationError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except CapacityError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except SvsimError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
