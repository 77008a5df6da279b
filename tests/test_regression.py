"""Datasets and encrypted regression against outputs of the reference
(encirc/datasets.py, encirc/regression.py) stored in tests/golden."""
import io
from fractions import Fraction

import pytest

from paper_2005_01945_b200 import PoolConfig, ReferenceEngine, WorkerPool
from paper_2005_01945_b200.datasets import (
    Dataset, DatasetFormatError, read_csv, synthesize, to_csv_text, write_csv,
)
from paper_2005_01945_b200.regression import SingularSystemError, fit_encrypted, solve_exact


def check_regression_against_reference(engine_factory, golden, kinds=("numerical", "binary")):
    for kind in kinds:
        rec = golden["meta"]["regression"][kind]
        ds = synthesize(kind, 12, 3, seed=4)
        assert to_csv_text(ds) == rec["csv"] and list(ds.coefficients) == rec["truth"]
        eng = engine_factory()
        rep = fit_encrypted(eng, ds, bits=12)
        assert [[c.numerator, c.denominator] for c in rep.coefficients] == rec["coefficients"]
        assert [list(r) for r in rep.gram] == rec["gram"] and list(rep.moment) == rec["moment"]
        assert rep.verified and [int(c) for c in rep.coefficients] == rec["truth"]
        assert eng.stats.as_record() == rec["stats"]


def test_regression_matches_reference(golden):
    check_regression_against_reference(
        lambda: ReferenceEngine(pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 22))), golden)


def test_csv_roundtrip_and_errors(tmp_path):
    ds = synthesize("binary", 6, 2, seed=1, noise=3)
    path = tmp_path / "d.csv"
    write_csv(str(path), ds)
    back = read_csv(str(path))
    assert back.rows == ds.rows and back.target == ds.target and back.kind == "binary"
    assert read_csv(io.StringIO("a,b,y\n1,2,3\n\n4,5,6\n7,8,9\n")).kind == "numerical"
    for text in ("", "y\n1\n", "a,y\n1\n", "a,y\nx,1\n"):
        with pytest.raises(DatasetFormatError):
            read_csv(io.StringIO(text))
    for bad in (lambda: synthesize("ordinal", 3, 1), lambda: synthesize("binary", 1, 2),
                lambda: synthesize("binary", 3, 2, coefficients=[1]), lambda: synthesize("binary", 3, 2, coefficients=[1, -1]),
                lambda: Dataset(("a",), ((200,),), (1,), "numerical"), lambda: Dataset(("a",), ((1,),), (-1,), "binary")):
        with pytest.raises(DatasetFormatError):
            bad()


def test_exact_solver_and_guards():
    assert solve_exact([[2, 1], [1, 3]], [3, 5]) == [Fraction(4, 5), Fraction(7, 5)]
    assert solve_exact([[0, 1], [1, 0]], [2, 3]) == [3, 2]
    with pytest.raises(SingularSystemError):
        solve_exact([[1, 2], [2, 4]], [1, 2])
    with pytest.raises(ValueError):
        solve_exact([[1, 2]], [1])
    ds = Dataset(("a",), ((100,), (100,)), (70000, 1), "numerical")
    with pytest.raises(ValueError):
        fit_encrypted(ReferenceEngine(), ds, bits=16)  # target does not fit
    with pytest.raises(ValueError):
        fit_encrypted(ReferenceEngine(), Dataset(("a",), ((120,),) * 300, (1,) * 300, "numerical"), bits=10)
