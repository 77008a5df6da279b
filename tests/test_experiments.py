"""The experiment harness and CLI against rows produced by the reference's own
harness (encirc/bench.py, encirc/cli.py) on its cleartext engine."""
import io
import json

import pytest

from paper_2005_01945_b200 import GateKind, PoolConfig, ReferenceEngine, WorkerPool, experiments
from paper_2005_01945_b200.cli import main


def harness_engine():
    return ReferenceEngine(pool=WorkerPool(PoolConfig(workers=1)), seed=3)


def test_rows_equal_the_reference_harness(golden):
    rows = []
    rows += experiments.bench_gate(harness_engine(), (4, 8, 16, 32), (GateKind.AND, GateKind.XOR))
    rows += experiments.bench_compound(harness_engine(), (1, 4, 8))
    rows += experiments.bench_add(harness_engine(), (16, 32), "bitwise", (1, 4))
    rows += experiments.bench_add(harness_engine(), (16,), "numberwise", (1,))
    rows += experiments.bench_mul(harness_engine(), (16,), "naive", (1, 4))
    rows += experiments.bench_mul(harness_engine(), (16,), "karatsuba", (1,))
    rows += experiments.bench_matmul(harness_engine(), (2, 4), "cannon")
    rows += experiments.bench_matmul(harness_engine(), (2,), "flat")
    assert [r.record(omit_timing=True) for r in rows] == golden["meta"]["harness_rows"]


def test_writers_and_schema():
    rows = experiments.bench_add(harness_engine(), (8,), "bitwise", (1,))
    buf = io.StringIO()
    experiments.write_csv(buf, rows, omit_timing=True)
    head, line = buf.getvalue().strip().split("\n")
    assert head == ",".join(experiments.RESULT_COLUMNS)
    assert line == "add-bitwise,8,1,reference,1,0.000000,8,16,40,24,true"
    buf = io.StringIO()
    experiments.write_jsonl(buf, rows, omit_timing=True)
    assert json.loads(buf.getvalue())["batch_launches"] == 24


def test_unsupported_requests_raise():
    eng = harness_engine()
    for bad in (lambda: experiments.bench_gate(eng, (1,)), lambda: experiments.bench_gate(eng, (128,)),
                lambda: experiments.bench_gate(eng, (4,), (GateKind.NOT,)),
                lambda: experiments.bench_add(eng, (8,), "carry-save"),
                lambda: experiments.bench_mul(eng, (12,), "karatsuba"),
                lambda: experiments.bench_matmul(eng, (3,)),
                lambda: experiments.bench_matmul(eng, (2,), "strassen")):
        with pytest.raises(experiments.UnsupportedWidthError):
            bad()


def test_cli_exit_codes_and_reproducible_rows(tmp_path, capsys):
    out1, out2 = tmp_path / "a.csv", tmp_path / "b.csv"
    base = ["add", "--engine", "reference", "--n", "8,16", "--ell", "1,4", "--seed", "5", "--workers", "1", "--omit-timing"]
    assert main(base + ["--out", str(out1)]) == 0
    assert main(base + ["--out", str(out2)]) == 0
    assert out1.read_bytes() == out2.read_bytes()
    assert out1.read_text().count("\n") == 5
    assert main(["mul", "--engine", "reference", "--algorithm", "karatsuba", "--n", "12"]) == 2
    assert main(["matmul", "--engine", "reference", "--rank", "16", "--algorithm", "flat"]) == 2  # 2**20 job ceiling
    assert main(["gate", "--engine", "reference", "--kinds", "nope"]) == 2
    assert main(["keygen", "--engine", "reference"]) == 2
    key = tmp_path / "k.bin"
    assert main(["keygen", "--out", str(key), "--seed", "4"]) == 0
    assert main(["gate", "--engine", "b200-tfhe", "--key", str(tmp_path / "missing.bin")]) == 2
    data = tmp_path / "d.csv"
    assert main(["dataset", "--rows", "8", "--attrs", "2", "--kind", "binary", "--seed", "2", "--out", str(data)]) == 0
    assert main(["linreg", str(data), "--engine", "reference", "--bits", "8", "--format", "json",
                 "--out", str(tmp_path / "l.json")]) == 0
    assert json.loads((tmp_path / "l.json").read_text())["experiment"] == "linreg-binary"
    singular = tmp_path / "s.csv"
    singular.write_text("a,b,y\n1,1,2\n1,1,2\n")
    assert main(["linreg", str(singular), "--engine", "reference", "--bits", "8"]) == 2
    capsys.readouterr()
