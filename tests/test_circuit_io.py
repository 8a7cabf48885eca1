"""Circuit text format vs the reference's own parser/formatter outputs
(tests/golden/circuit_io.json, made by make_golden.py from svsim)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, circuit_from_rows
from paper_1801_01037_b200 import ParseError
from paper_1801_01037_b200 import workloads as w
from paper_1801_01037_b200.circuit_io import format_circuit, parse_circuit


def golden():
    with open(os.path.join(GOLDEN, "circuit_io.json")) as fh:
        return json.load(fh)


def rows(c):
    return [[op.target, -1 if op.control is None else op.control, *op.gate.as_doubles()] for op in c.ops]


def test_parse_matches_reference():
    for case in golden()["parse"]:
        if "error_line" in case:
            with pytest.raises(ParseError) as exc:
                parse_circuit(case["text"])
            assert exc.value.line == case["error_line"], case["text"]
        else:
            c = parse_circuit(case["text"])
            assert c.n == case["n"]
            assert np.array_equal(np.array(rows(c)), np.array(case["ops"]))


def test_cli_parse_error_exit_code(tmp_path):
    from paper_1801_01037_b200.__main__ import main

    p = tmp_path / "bad.txt"
    p.write_text("qubits 2\nx 5\n")
    assert main(["run", str(p)]) == 2


@pytest.mark.gpu
def test_cli_run_matches_oracle(cuda_ok, tmp_path):
    import oracle
    from paper_1801_01037_b200.__main__ import main

    circ = w.random_layer_circuit(8, 4, seed=3)
    p = tmp_path / "c.txt"
    p.write_text(format_circuit(circ))
    a = np.zeros(256, np.complex128)
    a[0] = 1
    want = oracle.run_ops(a, w.oracle_ops(parse_circuit(p.read_text())))
    for extra in ([], ["--fused"], ["--ranks", "4", "--layout", "auto"]):
        out = tmp_path / "o.txt"
        assert main(["run", str(p), "--out", str(out)] + extra) == 0
        vals = np.array([complex(float(r), float(i)) for _, r, i in
                         (ln.split(",") for ln in out.read_text().splitlines())])
        assert np.max(np.abs(vals - want)) <= 1e-12, extra
    assert (tmp_path / "o.txt.stats.csv").read_text().startswith("gate_index,qubit")


def test_format_matches_reference_and_round_trips():
    for case in golden()["format"]:
        c = circuit_from_rows(case["n"], case["ops"])
        assert format_circuit(c) == case["text"]
        back = parse_circuit(case["text"])
        assert rows(back) == rows(c)
    c = w.random_layer_circuit(6, 3, seed=1)
    assert rows(parse_circuit(format_circuit(c))) == rows(c)
