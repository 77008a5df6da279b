"""Levelised (deferred) launch execution of GateEngine: a lazy engine counts and checks every launch at
the call, runs queued launches as one kernel launch when a result is needed, and must be
indistinguishable from the eager engine in results, ciphertext words, statistics and errors.
Exercised on CPU with the host oracle engine (real bootstraps by the C oracle, small LWE dimension)."""
import gc

import numpy as np
import pytest

from paper_2005_01945_b200 import (
    BootstrapMarginError, GateKind, LweParams, PoolConfig, WorkerPool, add_bitwise, decrypt_int, decrypt_vector,
    encrypt_int, encrypt_vector, keygen, mul_naive, vec_add,
)
from tests.host_engine import HostOracleEngine


@pytest.fixture(scope="module")
def small_key():
    return keygen(LweParams(m=20), seed=5)


def engines(key):
    pool = lambda: WorkerPool(PoolConfig(workers=1, max_batch=1 << 16))
    eager = HostOracleEngine(key, seed=3, pool=pool(), lazy=False)
    lazy = HostOracleEngine(key, seed=3, pool=pool(), lazy=True)
    lazy.eval_keys = eager.eval_keys
    return eager, lazy


def test_lazy_engine_is_indistinguishable_and_launches_less(small_key):
    eager, lazy = engines(small_key)
    outs = {}
    for eng in (eager, lazy):
        x, y = encrypt_int(eng, 0xB7, 8), encrypt_int(eng, 0x5D, 8)
        eng.reset_stats()
        eng.physical_launches = 0
        s = add_bitwise(x, y)
        p = mul_naive(encrypt_int(eng, 11, 4), encrypt_int(eng, 13, 4))
        v = vec_add(encrypt_vector(eng, [3, 200, 77], 8), encrypt_vector(eng, [250, 100, 9], 8))
        rec = eng.stats.as_record()
        words = eng.read_rows([b.row for b in s.bits] + [b.row for b in p.bits])
        outs[eng.lazy] = (decrypt_int(eng, s), decrypt_int(eng, p), decrypt_vector(eng, v), rec, words,
                          eng.physical_launches)
    e, l = outs[False], outs[True]
    assert e[0] == l[0] == (0xB7 + 0x5D) % 256 and e[1] == l[1] == 143 and e[2] == l[2] == [253, 44, 86]
    assert e[3] == l[3]                       # the reference's counters do not see the deferral
    assert np.array_equal(e[4], l[4])         # nor do the ciphertexts: a bootstrap draws no randomness
    assert e[5] == e[3]["batch_launches"]     # eager: one kernel launch per logical launch
    assert l[5] < 0.75 * e[5]                 # lazy: the carry-independent launches ride along


def test_adder_chain_is_two_kernel_launches_per_bit(small_key):
    _, lazy = engines(small_key)
    n = 6
    x, y = encrypt_int(lazy, 41, n), encrypt_int(lazy, 22, n)
    lazy.reset_stats()
    lazy.physical_launches = 0
    s = add_bitwise(x, y)
    assert lazy.stats.batch_launches == 3 * n
    assert decrypt_int(lazy, s) == 63
    assert lazy.physical_launches == 2 * n + 1


def test_multiplier_tree_runs_as_a_wavefront(small_key):
    """The adders of consecutive tree levels overlap: the dependent chain of an n-bit multiply is about
    one 2n-bit adder (2 kernel launches per bit) plus 2 per extra level, not one adder per level."""
    eager, lazy = engines(small_key)
    n = 8
    got = {}
    for eng in (eager, lazy):
        x, y = encrypt_int(eng, 201, n), encrypt_int(eng, 173, n)
        eng.reset_stats()
        eng.physical_launches = 0
        p = mul_naive(x, y)
        got[eng.lazy] = (decrypt_int(eng, p), eng.stats.as_record(), eng.physical_launches,
                         eng.read_rows([b.row for b in p.bits]))
    assert got[False][0] == got[True][0] == 201 * 173
    assert got[False][1] == got[True][1] and got[False][1]["batch_launches"] == 1 + 3 * 6 * n
    assert np.array_equal(got[False][3], got[True][3])
    assert got[False][2] == 1 + 3 * 6 * n            # eager: 145 kernel launches
    assert got[True][2] <= 2 * (2 * n) + 2 * 3 + 3   # lazy: one adder deep plus a few


def test_queue_is_flushed_at_its_capacity(small_key):
    _, lazy = engines(small_key)
    lazy.MAX_DEFERRED_GATES = 8
    bits = [lazy.encrypt(i & 1) for i in range(6)]
    outs = [lazy.eval_gate(GateKind.XOR, bits[i], bits[(i + 1) % 6]) for i in range(6)]  # independent launches
    outs2 = lazy.eval_gate_batch(GateKind.AND, outs, outs)                                # 6 more: over the cap
    assert lazy._deferred_gates <= 8
    assert [lazy.decrypt(b) for b in outs2] == [1] * 6


def test_rows_freed_while_a_launch_is_queued_are_not_recycled(small_key):
    _, lazy = engines(small_key)
    # inputs die right after the call, while the launch is still queued ...
    out = lazy.eval_gate(GateKind.AND, lazy.encrypt(1), lazy.encrypt(1))
    gc.collect()
    assert lazy._deferred and lazy._alloc.hold
    # ... and fresh allocations must not land on their rows before the launch has run
    fresh = [lazy.encrypt(0) for _ in range(8)]
    assert lazy.decrypt(out) == 1 and not lazy._deferred and not lazy._alloc.hold
    assert [lazy.decrypt(b) for b in fresh] == [0] * 8
    # a queued launch whose result is dropped still runs (or not) without disturbing later ones
    lazy.eval_gate(GateKind.XOR, lazy.encrypt(1), lazy.encrypt(0))
    gc.collect()
    keep = lazy.eval_gate(GateKind.OR, lazy.encrypt(0), lazy.encrypt(1))
    assert lazy.decrypt(keep) == 1


def test_not_bootstrap_and_margin_errors_with_queued_launches(small_key):
    eager, lazy = engines(small_key)
    for eng in (eager, lazy):
        a, b = eng.encrypt(1), eng.encrypt(0)
        g = eng.eval_gate(GateKind.NAND, a, b)            # queued on the lazy engine
        assert eng.decrypt(eng.eval_not(g)) == 0           # NOT reads the row: the queue runs first
        r = eng.bootstrap(eng.eval_gate(GateKind.OR, a, b))
        assert eng.decrypt(r) == 1 and r.noise_bound == eng.fresh_bound
        noisy = eng.eval_gate(GateKind.AND, a, a)
        eng._bounds[noisy.row] = 0.2                       # over-noised by hand, as the reference's tests do
        with pytest.raises(BootstrapMarginError):          # raised at the call, not when the queue runs
            eng.eval_gate(GateKind.AND, noisy, a)
        assert eng.decrypt(eng.eval_gate(GateKind.XOR, a, b)) == 1


class _EarlyStarter(HostOracleEngine):
    """A lazy host engine that hands the lowest queued level over every `every` recorded launches, the way
    B200Engine does while its device would otherwise idle."""

    every = 3

    def _early_start(self):
        self._seen = getattr(self, "_seen", 0) + 1
        if self._seen % self.every == 0 and self._deferred:
            self._run_next_level()


@pytest.mark.parametrize("every", [1, 2, 5, 17])
def test_early_start_is_unobservable(small_key, every):
    """Levels handed to the device while the circuit is still being recorded (absolute level numbering: a launch
    whose inputs are already evaluated joins the next level to run): results, ciphertext words, statistics and row
    recycling are those of the eager engine, and the dependent chain does not grow beyond the eager one."""
    pool = lambda: WorkerPool(PoolConfig(workers=1, max_batch=1 << 16))
    eager = HostOracleEngine(small_key, seed=3, pool=pool(), lazy=False)
    early = _EarlyStarter(small_key, seed=3, pool=pool(), lazy=True)
    early.every = every
    early.eval_keys = eager.eval_keys
    got = {}
    for eng in (eager, early):
        x, y = encrypt_int(eng, 0xC5, 8), encrypt_int(eng, 0x3B, 8)
        eng.reset_stats()
        eng.physical_launches = 0
        p = mul_naive(x, y)
        s = add_bitwise(x, y)
        gc.collect()
        v = vec_add(encrypt_vector(eng, [9, 130], 8), encrypt_vector(eng, [250, 7], 8))
        got[eng is early] = (decrypt_int(eng, p), decrypt_int(eng, s), decrypt_vector(eng, v), eng.stats.as_record(),
                             eng.read_rows([b.row for b in p.bits] + [b.row for b in s.bits]), eng.physical_launches)
        assert not eng._deferred and eng._depth_done == 0 and not eng._alloc.hold
    assert got[True][:4] == got[False][:4]
    assert got[False][0] == 0xC5 * 0x3B and got[False][1] == (0xC5 + 0x3B) % 256 and got[False][2] == [3, 137]
    assert np.array_equal(got[True][4], got[False][4])
    assert got[True][5] <= got[False][5]
