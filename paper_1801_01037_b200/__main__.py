"""Command line on the B200 engine, mirroring the reference CLI's `run` and
`bench` subcommands (pkg/src/svsim/cli.py:127-156, 206-247).

    python -m paper_1801_01037_b200 run circ.txt [--ranks P] [--scheme b]
        [--layout auto|none] [--out FILE] [--fused]
    python -m paper_1801_01037_b200 bench --qubits N [--ranks P] [--gate h] [--repeat R]

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


def cmd_bench(args) -> int:
    from . import engine
    from .core import Circuit, GateOp, standard_gate
    from .partition import PartitionPlan

    n, k = args.qubits, _k(args.ranks)
    plan = PartitionPlan(n, k)
    g = standard_gate(args.gate)
    ops = tuple(GateOp("single", g, q) for q in range(n) for _ in range(args.repeat))
    _, stats = engine.run_circuit(Circuit(n, ops), plan, _scheme(args.scheme))
    print(f"n={n} ranks={plan.p} scheme={args.scheme} gate={args.gate} repeat={args.repeat}")
    local, comm = [], []
    for q in range(n):
        times = [st.wall_time for st in stats if st.qubit == q]
        med = statistics.median(times)
        (comm if q >= n - k else local).append(med)
        print(f"qubit {q:3d}  median {med * 1e3:10.4f} ms  {'comm' if q >= n - k else 'local'}")
    if comm and local:
        print(f"T = {statistics.median(comm) / statistics.median(local):.6g}")
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
    b = sub.add_parser("bench")
    b.add_argument("--qubits", type=int, required=True)
    b.add_argument("--ranks", type=int, default=1)
    b.add_argument("--scheme", default="b")
    b.add_argument("--gate", default="h")
    b.add_argument("--repeat", type=int, default=3)
    args = ap.parse_args(argv)
    try:
        return cmd_run(args) if args.cmd == "run" else cmd_bench(args)
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
