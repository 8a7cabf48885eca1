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


def test_cli_verify_bad_gate_exit_2(tmp_path):
    from paper_1801_01037_b200.__main__ import main

    p = tmp_path / "bad.circ"
    p.write_text("qubits 1\nu 0 1 0 0 0 0 0 0 2\n")  # non-unitary (ref test_cli.py:221-226)
    assert main(["verify", str(p)]) == 2


@pytest.mark.gpu
def test_cli_verify(cuda_ok, tmp_path, capsys):
    from paper_1801_01037_b200.__main__ import main

    p = tmp_path / "r.circ"
    p.write_text(format_circuit(w.random_layer_circuit(8, 6, seed=62)))
    for extra in (["--ranks", "8", "--scheme", "a"], ["--ranks", "8", "--scheme", "b"],
                  ["--ranks", "8", "--scheme", "chunked:4"], ["--fused"]):
        capsys.readouterr()
        assert main(["verify", str(p)] + extra) == 0, extra
        out = capsys.readouterr().out
        assert out.startswith("max deviation = ")
        assert float(out.split("=")[1]) <= 1e-10
    i = tmp_path / "i.circ"
    i.write_text("qubits 1\ni 0\n")
    capsys.readouterr()
    assert main(["verify", str(i)]) == 0
    assert float(capsys.readouterr().out.split("=")[1]) == 0.0


@pytest.mark.gpu
def test_cli_bench_format(cuda_ok, capsys):
    from paper_1801_01037_b200.__main__ import main

    assert main(["bench", "--qubits", "4", "--ranks", "1", "--repeat", "2"]) == 0
    out = capsys.readouterr().out
    assert "c = no communication" in out and "T = n/a" in out
    rows = [ln.split(",") for ln in out[out.index("gate_index,"):].strip().splitlines()[1:]]
    assert len(rows) == 8
    assert all(r[3] == "false" and r[4] == "0" and r[5] == "0" for r in rows)
    assert main(["bench", "--qubits", "12", "--ranks", "4", "--scheme", "b", "--repeat", "3"]) == 0
    out = capsys.readouterr().out
    assert "c = 5.00" in out
    t = [ln for ln in out.splitlines() if ln.startswith("T = ")][0]
    assert float(t.split("=")[1]) > 0.0
    rows = [ln.split(",") for ln in out[out.index("gate_index,"):].strip().splitlines()[1:]]
    comm = [r for r in rows if r[3] == "true"]
    assert len(comm) == 2 * 3 and all(int(r[5]) == 16 * (1 << 10) for r in comm)  # 16*L bytes (scheme b)
