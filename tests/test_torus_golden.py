"""Host torus layer and the oracle port against vectors produced by the
reference itself (tests/golden/make_golden.py)."""
import hashlib

import numpy as np
import pytest

from oracle import encirc_port as port
from paper_2005_01945_b200 import (
    DecryptionUnreliableError, LweParams, LweSample, TorusElement, decrypt_bit, encrypt_bit, keygen,
    lwe_linear, phase, trivial_sample,
)
from paper_2005_01945_b200.engine import _GATES, TWO_INPUT_KINDS


def _words(s):
    return np.concatenate([s.a.astype(np.uint32), np.array([s.b], dtype=np.uint32)])


def test_keygen_matches_reference(golden, params):
    assert np.array_equal(keygen(params, seed=11).bits, golden["key11_bits"])
    assert np.array_equal(keygen(params, seed=2024).bits, golden["key2024_bits"])
    assert np.array_equal(port.keygen_bits(11), golden["key11_bits"])
    # SURVEY appendix A known answers
    assert golden["key11_bits"][:16].tolist() == [0, 0, 1, 0, 1, 1, 1, 0, 0, 0, 0, 1, 1, 0, 1, 0]
    assert int(golden["key11_bits"].sum()) == 249


def test_fresh_encryption_words_match_reference(golden, key):
    rng = np.random.default_rng((5, 0))
    rng_port = np.random.default_rng((5, 0))
    for bit, want, want_phase in zip(golden["enc5_bits"], golden["enc5_words"], golden["enc5_phase"]):
        c = encrypt_bit(key, int(bit), rng)
        assert np.array_equal(_words(c), want)
        assert phase(key, c).word == int(want_phase)
        assert decrypt_bit(key, c) == int(bit)
        assert c.noise_bound == key.params.fresh_noise_bound
        assert np.array_equal(port.encrypt(key.bits, int(bit), rng_port).words(), want)
    # appendix A: first draw of engine seed 5
    assert golden["enc5_words"][0][:3].tolist() == [2881021352, 3457461230, 97294837]
    assert int(golden["enc5_words"][0][-1]) == 1137079019


def test_gate_linear_forms_match_reference(golden, key):
    p = key.params
    c1 = LweSample(golden["enc5_words"][0][:-1], int(golden["enc5_words"][0][-1]), p.fresh_noise_bound, 32)
    c0 = LweSample(golden["enc5_words"][1][:-1], int(golden["enc5_words"][1][-1]), p.fresh_noise_bound, 32)
    from oracle import tfhe_oracle as orc

    for kid, kind in enumerate(TWO_INPUT_KINDS):
        cx, cy, off = _GATES[kind][1]
        got = lwe_linear([c1, c0], [cx, cy], off * p.mu)
        assert np.array_equal(_words(got), golden["linear_words"][kid])
        assert got.noise_bound == (abs(cx) + abs(cy)) * p.fresh_noise_bound
        # the C oracle's linear form (what the CUDA kernel is compared with)
        assert np.array_equal(orc.gate_linear(_words(c1), _words(c0), kid, p.mu.word), golden["linear_words"][kid])
        s1 = port.Sample(c1.a, c1.b, c1.noise_bound)
        s0 = port.Sample(c0.a, c0.b, c0.noise_bound)
        assert np.array_equal(port.linear([s1, s0], [cx, cy], (off * p.mu.word) % (1 << 32)).words(),
                              golden["linear_words"][kid])


def test_oracle_port_launch_matches_reference(golden, key):
    eng = port.OracleLweEngine(key.bits.astype(np.uint32), seed=5)
    xs = [eng.encrypt((i >> 1) & 1) for i in range(32)]
    ys = [eng.encrypt(i & 1) for i in range(32)]
    assert np.array_equal(np.stack([c.words() for c in xs]), golden["launch_x_words"])
    assert np.array_equal(np.stack([c.words() for c in ys]), golden["launch_y_words"])
    outs = eng.launch(golden["launch_kind_ids"], xs, ys)
    assert np.array_equal(np.stack([c.words() for c in outs]), golden["launch_out_words"])
    assert [eng.decrypt(c) for c in outs] == golden["launch_out_bits"].tolist()
    assert (eng.launches, eng.bootstraps) == (1, 32)
    # the expected bits are the truth tables
    want = [port.TRUTH[i // 4][i % 4] for i in range(32)]
    assert golden["launch_out_bits"].tolist() == want


def test_oracle_port_multi_block_launch_hash(golden, key):
    eng = port.OracleLweEngine(key.bits.astype(np.uint32), seed=77, max_batch=4096)
    xs = [eng.encrypt(i % 2) for i in range(600)]
    ys = [eng.encrypt((i // 2) % 2) for i in range(600)]
    got = eng.eval_gate_batch(2, xs, ys)  # NAND
    h = hashlib.sha256(b"".join(c.words().tobytes() for c in got)).hexdigest()
    assert h == golden["meta"]["nand600_seed77_sha256"]


def test_torus_element_laws_small_grid():
    w = 4
    els = [TorusElement(k, w) for k in range(1 << w)]
    zero = TorusElement(0, w)
    for a in els:
        assert a + zero == a and a - a == zero and -(-a) == a
        assert (3 * a).word == (3 * a.word) % 16
        for b in els:
            assert a + b == b + a
            assert (a - b) + b == a
    assert TorusElement.from_fraction(1, 8).word == 1 << 29
    assert TorusElement.from_fraction(1, 8).signed() == 0.125
    assert (5 * TorusElement.from_fraction(1, 8)).signed() == -0.375
    with pytest.raises(ValueError):
        TorusElement(1, 4) + TorusElement(1, 5)


def test_default_params_and_derived_words(params):
    assert (params.m, params.alpha, params.w) == (500, 2.0**-15, 32)
    assert params.mu.word == 1 << 29
    assert params.fresh_clamp_word == 1 << 27
    assert params.fresh_noise_bound == 2.0**-5
    assert params.message_word(1) == 1 << 29 and params.message_word(0) == (1 << 32) - (1 << 29)
    with pytest.raises(ValueError):
        LweParams(m=0)
    with pytest.raises(ValueError):
        LweParams(alpha=0.1)


def test_decrypt_ties_and_refusal(key):
    p = key.params
    zero_mask = np.zeros(p.m, dtype=np.uint32)
    assert decrypt_bit(key, LweSample(zero_mask, 0, 0.0, 32)) == 0  # tie at 0
    assert decrypt_bit(key, LweSample(zero_mask, p.half_word, 0.0, 32)) == 0  # tie at 1/2
    assert decrypt_bit(key, trivial_sample(p, 1)) == 1
    assert decrypt_bit(key, trivial_sample(p, 0)) == 0
    with pytest.raises(DecryptionUnreliableError):
        decrypt_bit(key, LweSample(zero_mask, p.mu.word, p.mu_float / 2, 32))
    with pytest.raises(ValueError):
        encrypt_bit(key, 2, np.random.default_rng(0))


def test_lwe_linear_is_linear(key):
    rng = np.random.default_rng(3)
    cs = [encrypt_bit(key, b, rng) for b in (1, 0, 1)]
    z = lwe_linear(cs, [2, -3, 1])
    want = (2 * phase(key, cs[0]).word - 3 * phase(key, cs[1]).word + phase(key, cs[2]).word) % (1 << 32)
    assert phase(key, z).word == want
    assert z.noise_bound == 6 * key.params.fresh_noise_bound
    with pytest.raises(ValueError):
        lwe_linear([], [])
