"""Key material, the exact CPU oracle, and the host emulation of kernel K1.

The reference has no bootstrapping key and no blind rotation, so
these tests pin the oracle the only ways available: (i) algebraic audits of the
keys under the secret keys, (ii) decrypted outputs and the reference's declared
post-gate noise bound 2**-5, (iii) agreement of two independent evaluations of
the external product (integer schoolbook vs double-precision FFT), and (iv) the
kernel's own arithmetic run on host threads against the oracle, bit for bit."""
import ctypes

import numpy as np
import pytest

from oracle import tfhe_oracle as orc
from paper_2005_01945_b200 import LweParams, encrypt_bit, generate_evaluation_keys, keygen
from paper_2005_01945_b200.engine import TWO_INPUT_KINDS, truth_table
from paper_2005_01945_b200.keys import RingParams, negacyclic_mul_binary


def pack(s):
    return np.concatenate([s.a, [s.b]]).astype(np.uint32)


def signed(word):
    return ((int(word) / 2**32) + 0.5) % 1.0 - 0.5


def test_negacyclic_mul_binary_exact():
    rng = np.random.default_rng(0)
    N = 64
    s = rng.integers(0, 2, size=N).astype(np.uint32)
    a = rng.integers(0, 1 << 32, size=(3, N), dtype=np.uint32)
    got = negacyclic_mul_binary(a, s)
    for r in range(3):
        assert np.array_equal(got[r], orc.negacyclic_mul_numpy(s.astype(np.int64), a[r]))


def test_keys_are_deterministic_and_shaped(key, eval_keys):
    again = generate_evaluation_keys(key, seed=11)
    assert np.array_equal(again.bk, eval_keys.bk) and np.array_equal(again.ksk, eval_keys.ksk)
    other = generate_evaluation_keys(key, seed=12)
    assert not np.array_equal(other.ring_key, eval_keys.ring_key)
    assert eval_keys.bk.shape == (250, 3, 4, 2, 1024) and eval_keys.ksk.shape == (1024, 8, 501)
    assert set(np.unique(eval_keys.ring_key)) <= {0, 1}
    with pytest.raises(ValueError):
        RingParams(k=2)
    with pytest.raises(ValueError):
        RingParams(N=1000)


def test_bootstrapping_key_rows_decrypt_to_gadget_times_message(key, eval_keys):
    """TRLWE row (p, lvl) of key j of pair m has phase  msg * 2^(32-(lvl+1)*bgbit) * [X^0 of component p]  + small
    noise, msg = s_2m, s_2m+1, s_2m * s_2m+1 for j = 0, 1, 2 (the unrolled bootstrapping key)."""
    ring = eval_keys.ring
    sprime = eval_keys.ring_key.view(np.uint32)
    for m in (0, 3, 249):
        s1, s2 = int(key.bits[2 * m]), int(key.bits[2 * m + 1])
        for j, msg in enumerate((s1, s2, s1 * s2)):
            for r in range(4):
                p_idx, lvl = divmod(r, ring.bk_l)
                a = eval_keys.bk[m, j, r, 0].view(np.uint32)
                b = eval_keys.bk[m, j, r, 1].view(np.uint32)
                ph = orc.ring_phase(a, b, sprime).astype(np.int64)
                gadget = msg << (32 - (lvl + 1) * ring.bk_bgbit)
                # message polynomial: component 1 (b) carries +gadget at X^0; component 0 (a) carries
                # gadget * (-s') after taking the phase b - a*s'
                want = np.zeros(1024, dtype=np.int64)
                if p_idx == 1:
                    want[0] = gadget
                else:
                    want = -(gadget * sprime.astype(np.int64))
                err = ((ph - want + 2**31) % 2**32) - 2**31
                assert np.abs(err).max() < 400  # 7.18e-9 * 2^32 = 31 -> 400 is ~13 sigma


def test_odd_dimension_pads_the_last_pair_with_a_zero_key_bit():
    p = LweParams(m=7)
    k = keygen(p, seed=3)
    ek = generate_evaluation_keys(k, seed=3)
    assert ek.bk.shape == (4, 3, 4, 2, 1024)
    sprime = ek.ring_key.view(np.uint32)
    for j, msg in enumerate((int(k.bits[6]), 0, 0)):  # s_7 = 0: keys 1 and 2 of the last pair encrypt 0
        ph = orc.ring_phase(ek.bk[3, j, 2, 0].view(np.uint32), ek.bk[3, j, 2, 1].view(np.uint32), sprime).astype(np.int64)
        want = np.zeros(1024, dtype=np.int64)
        want[0] = msg << (32 - ring_bgbit(ek))
        err = ((ph - want + 2**31) % 2**32) - 2**31
        assert np.abs(err).max() < 400


def ring_bgbit(ek):
    return ek.ring.bk_bgbit


def test_key_switching_key_rows_decrypt(key, eval_keys):
    ring = eval_keys.ring
    s = key.bits.astype(np.uint64)
    for i in (0, 5, 1023):
        for j in range(ring.ks_t):
            row = eval_keys.ksk[i, j].view(np.uint32).astype(np.uint64)
            ph = (int(row[-1]) - int((row[:-1] * s).sum())) % 2**32
            want = int(eval_keys.ring_key[i]) << (32 - (j + 1) * ring.ks_basebit)
            err = ((ph - want + 2**31) % 2**32) - 2**31
            assert abs(err) < 2**32 * key.params.alpha * 8


@pytest.fixture(scope="module")
def oracle_run(key, eval_keys):
    rng = np.random.default_rng((99, 0))
    K = 32
    bx = [(g >> 1) & 1 for g in range(K)]
    by = [g & 1 for g in range(K)]
    xs = np.stack([pack(encrypt_bit(key, b, rng)) for b in bx])
    ys = np.stack([pack(encrypt_bit(key, b, rng)) for b in by])
    kinds = np.array([(g // 4) % 8 for g in range(K)], dtype=np.uint8)
    out, ext, bar = orc.gate_bootstrap_batch(xs, ys, kinds, key.params.mu.word, eval_keys.bk, eval_keys.ksk,
                                             fft=True, want_ext=True, want_bar=True)
    return dict(xs=xs, ys=ys, kinds=kinds, bx=bx, by=by, out=out, ext=ext, bar=bar)


def test_oracle_outputs_decrypt_to_truth_tables_within_fresh_bound(key, eval_keys, oracle_run):
    mu, bound = key.params.mu_float, key.params.fresh_noise_bound
    for g in range(len(oracle_run["kinds"])):
        want = truth_table(TWO_INPUT_KINDS[int(oracle_run["kinds"][g])])[(oracle_run["bx"][g] << 1) | oracle_run["by"][g]]
        ph = signed(orc.lwe_phase(oracle_run["out"][g], key.bits))
        assert (1 if ph > 0 else 0) == want
        assert abs(ph - (mu if want else -mu)) < bound  # reference invariant: encirc/torus.py:177-184
        # the extracted sample (before key switching) under the ring key is tighter still
        phe = signed(orc.lwe_phase(oracle_run["ext"][g], eval_keys.ring_key.view(np.uint32)))
        assert abs(phe - (mu if want else -mu)) < bound / 2


def test_oracle_exact_path_equals_fft_path(key, eval_keys, oracle_run):
    sel = slice(0, 6)
    out, ext = orc.gate_bootstrap_batch(oracle_run["xs"][sel], oracle_run["ys"][sel], oracle_run["kinds"][sel],
                                        key.params.mu.word, eval_keys.bk, eval_keys.ksk, fft=False, want_ext=True)
    assert np.array_equal(out, oracle_run["out"][sel])
    assert np.array_equal(ext, oracle_run["ext"][sel])


def test_oracle_mod_switch_and_trivial_inputs(key, eval_keys):
    p = key.params
    triv1 = np.zeros(501, dtype=np.uint32); triv1[-1] = p.message_word(1)
    triv0 = np.zeros(501, dtype=np.uint32); triv0[-1] = p.message_word(0)
    xs = np.stack([triv1, triv1, triv0, triv0])
    ys = np.stack([triv1, triv0, triv1, triv0])
    for kid, kind in enumerate(TWO_INPUT_KINDS):
        out, bar = orc.gate_bootstrap_batch(xs, ys, np.full(4, kid, np.uint8), p.mu.word, eval_keys.bk,
                                            eval_keys.ksk, want_bar=True)
        assert not bar[:, :-1].any()  # zero masks switch to zero rotations
        for g in range(4):
            want = truth_table(kind)[((1 - g // 2) << 1) | (1 - g % 2)]
            assert not out[g, :-1].any()  # a trivial input pair gives a trivial output
            assert int(out[g, -1]) == p.message_word(want)


def test_key_switch_digits_recompose():
    rng = np.random.default_rng(5)
    a = rng.integers(0, 1 << 32, size=1000, dtype=np.uint32).astype(np.int64)
    bias = (1 << 15) + sum(2 << (32 - 2 * (j + 1)) for j in range(8))
    ab = (a + bias) % 2**32
    rec = np.zeros_like(a)
    for j in range(8):
        d = ((ab >> (32 - 2 * (j + 1))) & 3) - 2
        assert d.min() >= -2 and d.max() <= 1
        rec += d << (32 - 2 * (j + 1))
    err = ((rec - a + 2**31) % 2**32) - 2**31
    assert np.abs(err).max() <= 1 << 15


@pytest.mark.parametrize("n", [12, 7])
def test_kernel_arithmetic_on_host_threads_matches_oracle(emu_lib, n):
    """The exact __host__ __device__ code of the K1 kernels (forward/inverse FFT, spectral rotation factors, key
    combination, decomposition, sample extract), driven by host threads, against the integer oracle: K1d (one
    ciphertext per warp, 32 threads) and K1e (one ciphertext over two CTAs of two 64-thread groups, 256 threads).
    Small LWE dimensions (even and odd: the padded last pair) keep it to seconds; the ring side is the production one."""
    p = LweParams(m=n)
    k = keygen(p, seed=3)
    ek = generate_evaluation_keys(k, seed=3)
    rng = np.random.default_rng(8)
    K = 6
    xs = np.stack([pack(encrypt_bit(k, g & 1, rng)) for g in range(K)])
    ys = np.stack([pack(encrypt_bit(k, (g >> 1) & 1, rng)) for g in range(K)])
    kinds = np.array([0, 4, 2, 7, 5, 8], dtype=np.uint8)
    out, ext = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, ek.bk, ek.ksk, want_ext=True)
    pairs = (n + 1) // 2
    vp = ctypes.c_void_p
    # K1e: chunks [pair][p][lvl][half][k4][key][c][t]
    bkf = np.empty((pairs, 2, 2, 2, 4, 3, 2, 64, 2), dtype=np.float64)
    emu_lib.emu_bk_transform(vp(ek.bk.ctypes.data), n, vp(bkf.ctypes.data))
    got = np.empty((K, 1025), dtype=np.uint32)
    emu_lib.emu_pair_gate_bootstrap(vp(xs.ctypes.data), vp(ys.ctypes.data), vp(kinds.ctypes.data), ctypes.c_int64(K), n,
                                    ctypes.c_uint32(p.mu.word), vp(bkf.ctypes.data), vp(got.ctypes.data))
    assert np.array_equal(got, ext)
    # K1d: chunks [pair][stage][qc][q4][key][c][lane]
    bkw = np.empty((pairs, 4, 4, 4, 3, 2, 32, 2), dtype=np.float64)
    emu_lib.emu_w_bk_transform(vp(ek.bk.ctypes.data), n, vp(bkw.ctypes.data))
    warp = np.empty((K, 1025), dtype=np.uint32)
    emu_lib.emu_w_gate_bootstrap(vp(xs.ctypes.data), vp(ys.ctypes.data), vp(kinds.ctypes.data), ctypes.c_int64(K), n,
                                 ctypes.c_uint32(p.mu.word), vp(bkw.ctypes.data), vp(warp.ctypes.data))
    assert np.array_equal(warp, ext)
    # a gate on trivial inputs (every rotation zero) skips every step in both kernels
    triv = np.zeros((2, n + 1), dtype=np.uint32)
    triv[:, n] = [p.message_word(1), p.message_word(0)]
    tk = np.array([2, 2], dtype=np.uint8)
    _, text = orc.gate_bootstrap_batch(triv, triv[::-1].copy(), tk, p.mu.word, ek.bk, ek.ksk, want_ext=True)
    for fn, key_arr in ((emu_lib.emu_pair_gate_bootstrap, bkf), (emu_lib.emu_w_gate_bootstrap, bkw)):
        tg = np.empty((2, 1025), dtype=np.uint32)
        fn(vp(triv.ctypes.data), vp(triv[::-1].copy().ctypes.data), vp(tk.ctypes.data), ctypes.c_int64(2), n,
           ctypes.c_uint32(p.mu.word), vp(key_arr.ctypes.data), vp(tg.ctypes.data))
        assert np.array_equal(tg, text)
    # K2's digit extraction against the oracle's key switch
    digits = np.empty((1024, 8), dtype=np.int32)
    emu_lib.emu_ks_digits(vp(ext[0].ctypes.data), vp(digits.ctypes.data))
    ks = np.zeros(n + 1, dtype=np.uint32)
    ks[n] = ext[0][1024]
    ks -= (digits.reshape(-1, 1).astype(np.uint32) * ek.ksk.reshape(-1, n + 1).view(np.uint32)).sum(axis=0, dtype=np.uint32)
    assert np.array_equal(ks, out[0])


def test_kernel_fft_roundtrip_and_spectrum(emu_lib):
    rng = np.random.default_rng(1)
    poly = rng.integers(-2**31, 2**31, size=1024).astype(np.int32)
    spec = np.empty((512, 2), dtype=np.float64)
    vp = ctypes.c_void_p
    emu_lib.emu_fft_forward(vp(poly.ctypes.data), vp(spec.ctypes.data))
    tw = np.exp(1j * np.pi * np.arange(512) / 1024)
    want = np.fft.ifft((poly[:512] + 1j * poly[512:]) * tw) * 512
    got = spec[:, 0] + 1j * spec[:, 1]
    assert np.abs(got - want).max() / np.abs(want).max() < 1e-14
    back = np.empty(1024, dtype=np.uint32)
    emu_lib.emu_fft_inverse(vp(spec.ctypes.data), vp(back.ctypes.data))
    assert np.array_equal(back.view(np.int32), poly)
    # the warp-level transform of K1d (16 points per lane, one exchange + one shuffle stage)
    spec_w = np.empty((512, 2), dtype=np.float64)
    emu_lib.emu_w_fft_forward(vp(poly.ctypes.data), vp(spec_w.ctypes.data))
    got_w = spec_w[:, 0] + 1j * spec_w[:, 1]
    assert np.abs(got_w - want).max() / np.abs(want).max() < 1e-14
    back_w = np.empty(1024, dtype=np.uint32)
    emu_lib.emu_w_fft_inverse(vp(spec_w.ctypes.data), vp(back_w.ctypes.data))
    assert np.array_equal(back_w.view(np.int32), poly)
