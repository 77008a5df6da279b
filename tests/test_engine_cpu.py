"""Engine contract on the cleartext engine (runs without a GPU).  The same
assertions run against B200Engine in tests/test_gpu_engine.py."""
import numpy as np
import pytest

from paper_2005_01945_b200 import (
    TWO_INPUT_KINDS, BootstrapMarginError, DecryptionUnreliableError, EncBit, GateKind, GateStats,
    LweParams, PoolConfig, ReferenceEngine, WorkerPool, truth_table,
)
from fractions import Fraction


def check_truth_tables(eng):
    for kind in TWO_INPUT_KINDS:
        for x in (0, 1):
            for y in (0, 1):
                out = eng.eval_gate(kind, eng.encrypt(x), eng.encrypt(y))
                assert eng.decrypt(out) == truth_table(kind)[(x << 1) | y], (kind, x, y)
    for x in (0, 1):
        assert eng.decrypt(eng.eval_not(eng.encrypt(x))) == 1 - x
        assert eng.decrypt(eng.eval_gate(GateKind.NOT, eng.trivial_bit(x))) == 1 - x


def check_not_is_free(eng):
    x = eng.encrypt(1)
    before = eng.snapshot_stats()
    y = eng.eval_not(x)
    d = eng.snapshot_stats().delta(before)
    assert (d.not_gates, d.bootstraps, d.batch_launches) == (1, 0, 0)
    assert y.noise_bound == x.noise_bound


def check_compound_economy(eng):
    x, y = eng.encrypt(1), eng.encrypt(0)
    before = eng.snapshot_stats()
    s, g = eng.eval_compound(GateKind.XOR, GateKind.AND, x, y)
    d = eng.snapshot_stats().delta(before)
    assert (d.compound_gates, d.single_gates, d.bootstraps, d.batch_launches) == (1, 0, 2, 1)
    assert (eng.decrypt(s), eng.decrypt(g)) == (1, 0)
    before = eng.snapshot_stats()
    eng.eval_gate(GateKind.XOR, x, y)
    eng.eval_gate(GateKind.AND, x, y)
    d = eng.snapshot_stats().delta(before)
    assert (d.single_gates, d.bootstraps, d.batch_launches) == (2, 2, 2)


def check_fresh_bound_and_bootstrap(eng):
    out = eng.eval_gate(GateKind.OR, eng.encrypt(0), eng.encrypt(1))
    assert out.noise_bound == eng.fresh_bound == 2.0**-5
    x = eng.encrypt(1)
    before = eng.snapshot_stats()
    y = eng.bootstrap(x)
    d = eng.snapshot_stats().delta(before)
    assert (d.bootstraps, d.batch_launches) == (1, 1)
    assert y.noise_bound == eng.fresh_bound and eng.decrypt(y) == 1
    assert eng.trivial_bit(1).noise_bound == 0.0


def check_argument_errors(eng):
    other = ReferenceEngine()
    with pytest.raises(ValueError):
        eng.eval_gate(GateKind.AND, eng.encrypt(1), other.encrypt(1))
    with pytest.raises(ValueError):
        eng.eval_gate(GateKind.AND, eng.encrypt(1))
    with pytest.raises(ValueError):
        eng.eval_gate(GateKind.NOT, eng.encrypt(1), eng.encrypt(1))
    with pytest.raises(ValueError):
        eng.eval_gate_batch(GateKind.AND, [], [])
    with pytest.raises(ValueError):
        eng.eval_gate_batch(GateKind.AND, [eng.encrypt(1)], [])
    with pytest.raises(ValueError):
        eng.eval_gate_batch(GateKind.NOT, [eng.encrypt(1)], [eng.encrypt(1)])
    with pytest.raises(ValueError):
        eng.encrypt(2)
    with pytest.raises(ValueError):
        eng.trivial_bit(-1)


def test_truth_tables(ref):
    check_truth_tables(ref)


def test_not_is_free(ref):
    check_not_is_free(ref)


def test_compound_economy(ref):
    check_compound_economy(ref)


def test_fresh_bound_and_bootstrap(ref):
    check_fresh_bound_and_bootstrap(ref)


def test_argument_errors(ref):
    check_argument_errors(ref)


def test_margins_match_reference(ref, golden):
    for kind in TWO_INPUT_KINDS:
        assert ref.gate_margin(kind) == golden["meta"]["margins"][kind.value]
    assert ref.fresh_bound == golden["meta"]["fresh_bound"]


def test_margin_and_decrypt_refusal(ref):
    mu = ref.params.mu_float
    with pytest.raises(BootstrapMarginError):
        ref.eval_gate(GateKind.AND, EncBit(ref, clear=1, bound=mu), ref.encrypt(1))
    nearly = EncBit(ref, clear=1, bound=0.9 * mu)
    ref.eval_gate(GateKind.AND, nearly, ref.trivial_bit(1))
    with pytest.raises(BootstrapMarginError):
        ref.eval_gate(GateKind.XOR, nearly, nearly)
    with pytest.raises(BootstrapMarginError):
        ref.bootstrap(EncBit(ref, clear=1, bound=mu))
    with pytest.raises(DecryptionUnreliableError):
        ref.decrypt(EncBit(ref, clear=1, bound=mu / 2))


def test_boundary_mu_rejected_at_build():
    with pytest.raises(ValueError):
        ReferenceEngine(LweParams(alpha=0.0, mu=Fraction(1, 4)))


def test_batch_split_at_max_batch():
    eng = ReferenceEngine(pool=WorkerPool(PoolConfig(workers=1, max_batch=8)))
    xs = [eng.encrypt(i & 1) for i in range(20)]
    outs = eng.eval_gate_batch(GateKind.NAND, xs, xs)
    assert [eng.decrypt(o) for o in outs] == [1 - (i & 1) for i in range(20)]
    st = eng.snapshot_stats()
    assert (st.batch_launches, st.largest_batch, st.bootstraps, st.single_gates) == (3, 8, 20, 20)


def test_stats_record_and_delta():
    a = GateStats(single_gates=3, bootstraps=5, batch_launches=2, largest_batch=4)
    b = a.snapshot()
    b.single_gates += 2
    b.largest_batch = 9
    d = b.delta(a)
    assert (d.single_gates, d.bootstraps, d.largest_batch) == (2, 0, 9)
    assert set(a.as_record()) == {"single_gates", "compound_gates", "not_gates", "bootstraps", "batch_launches", "largest_batch"}
    b.reset()
    assert b == GateStats()


def test_rows_are_recycled(ref):
    top0 = ref._alloc.top
    for _ in range(50):
        xs = [ref.encrypt(1) for _ in range(8)]
        ref.eval_gate_batch(GateKind.AND, xs, xs)
        del xs
    assert ref._alloc.top <= top0 + 64
