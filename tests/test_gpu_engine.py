"""B200Engine behind the reference's GateEngine API: the engine-contract checks
of tests/test_engine_cpu.py re-run on the GPU engine, golden vectors of the
reference, circuits against native arithmetic with the reference's counts."""
import numpy as np
import pytest

from paper_2005_01945_b200 import (
    BootstrapMarginError, EncBit, GateKind, LweSample, PoolConfig, WorkerPool, add_bitwise, decrypt_int,
    decrypt_matrix, decrypt_vector, encrypt_int, encrypt_matrix, encrypt_vector, mat_mul_cannon,
    mat_mul_flat, mul_karatsuba, mul_naive, vec_add, vec_mul,
)
from tests.test_circuits_cpu import check_scalar_circuits_against_reference
from tests.test_engine_cpu import (
    check_argument_errors, check_compound_economy, check_fresh_bound_and_bootstrap, check_not_is_free,
    check_truth_tables,
)

pytestmark = pytest.mark.gpu


def test_native_library_is_loaded(b200):
    import ctypes

    from paper_2005_01945_b200 import _cabi

    assert isinstance(_cabi.lib(), ctypes.CDLL)
    assert b200.kernel_launches >= 2  # key setup ran on the device


def test_engine_contract(b200):
    check_truth_tables(b200)
    check_not_is_free(b200)
    check_compound_economy(b200)
    check_fresh_bound_and_bootstrap(b200)
    check_argument_errors(b200)


def test_fresh_ciphertexts_are_the_references(key, eval_keys, golden):
    """Engine seed 5: the first encryptions are word-for-word the reference's
    (encirc/engine.py:424,429-430)."""
    from paper_2005_01945_b200 import B200Engine

    eng = B200Engine(key, seed=5, eval_keys=eval_keys)
    bits = [eng.encrypt(int(b)) for b in golden["enc5_bits"]]
    for bit, want in zip(bits, golden["enc5_words"]):
        s = bit.sample
        assert np.array_equal(s.a, want[:-1]) and s.b == int(want[-1])
        assert s.noise_bound == eng.fresh_bound and s.w == 32
    assert [eng.decrypt(b) for b in bits] == golden["enc5_bits"].tolist()
    # the reference's oracle launch on the same inputs decrypts to the same bits
    eng = B200Engine(key, seed=5, eval_keys=eval_keys)
    xs = [eng.encrypt((i >> 1) & 1) for i in range(32)]
    ys = [eng.encrypt(i & 1) for i in range(32)]
    from paper_2005_01945_b200.engine import TWO_INPUT_KINDS
    from paper_2005_01945_b200 import JobBatch

    outs = eng.pool.execute_batch(JobBatch([TWO_INPUT_KINDS[i // 4] for i in range(32)], xs, ys), eng)
    assert [eng.decrypt(c) for c in outs] == golden["launch_out_bits"].tolist()
    assert np.array_equal(np.stack([np.append(c.sample.a, c.sample.b) for c in xs]), golden["launch_x_words"])


def test_margin_errors_and_adopted_samples(b200):
    mu = b200.params.mu_float
    good = b200.encrypt(1)
    s = good.sample
    bad = EncBit(b200, sample=LweSample(s.a, s.b, mu, 32))
    with pytest.raises(BootstrapMarginError):
        b200.eval_gate(GateKind.AND, bad, b200.encrypt(1))
    with pytest.raises(BootstrapMarginError):
        b200.bootstrap(bad)
    ok = EncBit(b200, sample=LweSample(s.a, s.b, s.noise_bound, 32))
    assert b200.decrypt(b200.eval_gate(GateKind.AND, ok, good)) == 1


def test_same_seed_same_ciphertexts_and_worker_independence(key, eval_keys):
    from paper_2005_01945_b200 import B200Engine

    outs = []
    for workers in (1, 8):
        eng = B200Engine(key, seed=77, pool=WorkerPool(PoolConfig(workers=workers)), eval_keys=eval_keys)
        xs = [eng.encrypt(i % 2) for i in range(300)]
        ys = [eng.encrypt((i // 2) % 2) for i in range(300)]
        got = eng.eval_gate_batch(GateKind.NAND, xs, ys)
        assert eng.snapshot_stats().batch_launches == 1
        outs.append(eng.read_rows([b.row for b in got]).tobytes())
        assert [eng.decrypt(b) for b in got] == [1 - ((i % 2) & ((i // 2) % 2)) for i in range(300)]
    assert outs[0] == outs[1]


def test_scalar_circuits_counts_and_results(b200, golden):
    check_scalar_circuits_against_reference(b200, golden, widths=(8, 16))


def test_random_circuits_agree_with_cleartext_engine(b200):
    from paper_2005_01945_b200 import ReferenceEngine
    from paper_2005_01945_b200.engine import TWO_INPUT_KINDS

    rng = np.random.default_rng(5)
    for trial in range(6):
        ref = ReferenceEngine(b200.params)
        engines = (ref, b200)
        for e in engines:
            e.reset_stats()
        inputs = rng.integers(0, 2, size=6).tolist()
        wires = [[e.encrypt(v) for v in inputs] for e in engines]
        for _ in range(20):
            op = rng.integers(0, 3)
            i, j = rng.integers(0, len(wires[0]), size=2)
            ka, kb = (TWO_INPUT_KINDS[t] for t in rng.integers(0, 8, size=2))
            for e, w in zip(engines, wires):
                if op == 0:
                    w.append(e.eval_gate(ka, w[i], w[j]))
                elif op == 1:
                    w.extend(e.eval_compound(ka, kb, w[i], w[j]))
                else:
                    w.append(e.eval_not(w[i]))
        assert [ref.decrypt(b) for b in wires[0]] == [b200.decrypt(b) for b in wires[1]]
        assert ref.stats.as_record() == b200.stats.as_record()


def test_arithmetic_16_and_32_bit(b200):
    rng = np.random.default_rng((11, 2))
    for n in (16, 32):
        a, b = int(rng.integers(0, 1 << n, dtype=np.uint64)), int(rng.integers(0, 1 << n, dtype=np.uint64))
        x, y = encrypt_int(b200, a, n), encrypt_int(b200, b, n)
        b200.reset_stats()
        assert decrypt_int(b200, add_bitwise(x, y)) == (a + b) % (1 << n)
        assert (b200.stats.bootstraps, b200.stats.batch_launches) == (5 * n, 3 * n)
        b200.reset_stats()
        assert decrypt_int(b200, mul_naive(x, y)) == a * b
        assert b200.stats.bootstraps == 11 * n * n - 10 * n
    a, b = 40503, 65535
    x, y = encrypt_int(b200, a, 16), encrypt_int(b200, b, 16)
    assert decrypt_int(b200, mul_karatsuba(x, y)) == a * b


def test_vectors_and_matrices(b200):
    rng = np.random.default_rng(21)
    u = rng.integers(0, 1 << 16, size=24).tolist()
    v = rng.integers(0, 1 << 16, size=24).tolist()
    eu, ev = encrypt_vector(b200, u, 16), encrypt_vector(b200, v, 16)
    b200.reset_stats()
    assert decrypt_vector(b200, vec_add(eu, ev)) == [(a + b) % (1 << 16) for a, b in zip(u, v)]
    assert b200.stats.batch_launches == 48
    assert decrypt_vector(b200, vec_mul(eu, ev)) == [a * b for a, b in zip(u, v)]
    A = rng.integers(0, 1 << 16, size=(3, 3)).tolist()
    B = rng.integers(0, 1 << 16, size=(3, 3)).tolist()
    want = [[sum(A[i][t] * B[t][j] for t in range(3)) % (1 << 16) for j in range(3)] for i in range(3)]
    ea, eb = encrypt_matrix(b200, A, 16), encrypt_matrix(b200, B, 16)
    assert decrypt_matrix(b200, mat_mul_flat(ea, eb)) == want
    assert decrypt_matrix(b200, mat_mul_cannon(ea, eb)) == want


def test_noise_hygiene_over_many_gate_outputs(b200):
    """10,000 chained gate outputs: all decrypt correctly and every phase stays
    within the declared fresh bound of +-mu (reference acceptance :328-374)."""
    rng = np.random.default_rng(9)
    bits = rng.integers(0, 2, size=2500)
    rows, own = b200.encrypt_rows(bits.tolist())
    clear = bits.copy()
    seen = 0
    for step in range(4):
        perm = rng.permutation(len(rows))
        kind = (GateKind.NAND, GateKind.XOR, GateKind.ORNY, GateKind.XNOR)[step]
        out, own2 = b200.gate_rows(kind, rows, rows[perm])
        from paper_2005_01945_b200 import truth_table

        tt = np.array(truth_table(kind))
        clear = tt[(clear << 1) | clear[perm]]
        ph = b200.phases(out).astype(np.int64)
        target = np.where(clear == 1, 1 << 29, (1 << 32) - (1 << 29))
        err = ((ph - target + 2**31) % 2**32) - 2**31
        assert np.abs(err).max() < (1 << 27)
        assert np.array_equal(b200.decrypt_rows(out), clear)
        rows, own = out, own2
        seen += len(out)
    assert seen == 10000


def test_wire_formats_on_device_ciphertexts(key, eval_keys, golden):
    """Engine seed 9: device-resident integers serialise to the reference's bytes and load back."""
    from paper_2005_01945_b200 import B200Engine, dump_int, dump_matrix, dump_vector, load_int, load_matrix, load_vector

    eng = B200Engine(key, seed=9, eval_keys=eval_keys)
    x = encrypt_int(eng, 11, 4)
    vec = encrypt_vector(eng, [3, 5], 3)
    mat = encrypt_matrix(eng, [[1, 2], [3, 0]], 2)
    assert dump_int(x) == golden["ser_int"].tobytes()
    assert dump_vector(vec) == golden["ser_vector"].tobytes()
    assert dump_matrix(mat) == golden["ser_matrix"].tobytes()
    y = load_int(golden["ser_int"].tobytes(), eng)
    assert decrypt_int(eng, add_bitwise(x, y)) == (11 + 11) % 16
    assert decrypt_vector(eng, load_vector(dump_vector(vec_add(vec, vec)), eng)) == [6, 2]
    assert decrypt_matrix(eng, load_matrix(golden["ser_matrix"].tobytes(), eng)) == [[1, 2], [3, 0]]


def test_cli_runs_the_reference_experiments_on_the_gpu(tmp_path, golden):
    import json

    from paper_2005_01945_b200.cli import main

    out = tmp_path / "rows.json"
    assert main(["add", "--engine", "b200-tfhe", "--n", "16", "--ell", "1,4", "--seed", "3", "--workers", "1",
                 "--format", "json", "--omit-timing", "--out", str(out)]) == 0
    rows = [json.loads(line) for line in out.read_text().splitlines()]
    want = [r for r in golden["meta"]["harness_rows"] if r["experiment"] in ("add-bitwise", "vec-add") and r["n"] == 16]
    assert len(rows) == len(want) == 2
    for got, ref in zip(rows, want):
        assert got["engine"] == "b200-tfhe" and got["correct"] is True
        for field in ("experiment", "n", "ell_or_rank", "workers", "single_gates", "compound_gates", "bootstraps",
                      "batch_launches"):
            assert got[field] == ref[field]
    assert main(["gate", "--engine", "b200-tfhe", "--sizes", "4,300", "--max-size", "512", "--kinds", "nand,xor",
                 "--seed", "3", "--out", str(tmp_path / "g.csv")]) == 0
    assert main(["compound", "--engine", "b200-tfhe", "--sizes", "1,8", "--seed", "3", "--out", str(tmp_path / "c.csv")]) == 0


def test_encrypted_regression_on_the_gpu(key, eval_keys, golden):
    from paper_2005_01945_b200 import B200Engine
    from tests.test_regression import check_regression_against_reference

    check_regression_against_reference(
        lambda: B200Engine(key, seed=3, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 22)), eval_keys=eval_keys),
        golden)


def test_lazy_and_eager_execution_agree_on_the_device(key, eval_keys):
    """Levelised (recorded, level-by-level) execution against one kernel sequence per logical launch, on the real
    device row pool with its quarantine / recycling: identical ciphertext words, results and GateStats for a 16-bit
    multiply and a 4 x 4 Cannon matrix product (tests/test_lazy_engine.py checks the same on the host stand-in)."""
    from paper_2005_01945_b200 import B200Engine

    rng = np.random.default_rng(41)
    a, b = (int(v) for v in rng.integers(0, 1 << 16, size=2))
    A, Bm = (rng.integers(0, 1 << 6, size=(4, 4)).tolist() for _ in range(2))
    seen = {}
    for mode in ("lazy", "eager"):
        eng = B200Engine(key, seed=23, eval_keys=eval_keys, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)),
                         initial_rows=1 << 12)  # small pool: growth and row recycling happen during the run
        eng.lazy = mode == "lazy"
        prod = mul_naive(encrypt_int(eng, a, 16), encrypt_int(eng, b, 16))
        mat = mat_mul_cannon(encrypt_matrix(eng, A, 6), encrypt_matrix(eng, Bm, 6))
        words = np.concatenate([eng.read_rows(prod._rows)] + [eng.read_rows(c._rows) for c in mat.data])
        assert decrypt_int(eng, prod) == a * b
        assert decrypt_matrix(eng, mat) == [[sum(A[i][t] * Bm[t][j] for t in range(4)) % 64 for j in range(4)]
                                            for i in range(4)]
        seen[mode] = (words, eng.stats.as_record(), eng.physical_launches)
    assert np.array_equal(seen["lazy"][0], seen["eager"][0])
    assert seen["lazy"][1] == seen["eager"][1]
    assert seen["lazy"][2] < seen["eager"][2]  # fewer kernel-launch levels than logical launches


def test_device_side_encryption(key, eval_keys):
    """tfb_rows_encrypt: every row decrypts to its bit, the noise is the rounded clipped Gaussian(alpha) of the
    reference's fresh encryption (encirc/torus.py:233-271), the stream is deterministic in (seed, call order), and
    the config-5 input volume (2 x 4096 x 32 bits) is produced well inside half a second."""
    import time

    from paper_2005_01945_b200 import B200Engine

    eng = B200Engine(key, seed=9, eval_keys=eval_keys, device_encrypt=True)
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2, size=1 << 16)
    rows, owner = eng.encrypt_rows(bits)
    assert np.array_equal(eng.decrypt_rows(rows), bits)
    ph = eng.phases(rows).astype(np.int64)
    target = np.where(bits == 1, 1 << 29, (1 << 32) - (1 << 29))
    err = ((ph - target + 2**31) % 2**32) - 2**31
    sigma = key.params.alpha * 2.0**32
    assert abs(err.std() / sigma - 1.0) < 0.02 and abs(err.mean()) < 4 * sigma / np.sqrt(len(err))
    assert np.abs(err).max() < (1 << 27)
    # rounded Gaussian: about 68.3 % / 95.4 % inside one / two sigma
    assert abs((np.abs(err) < sigma).mean() - 0.6827) < 0.01 and abs((np.abs(err) < 2 * sigma).mean() - 0.9545) < 0.005
    words = eng.read_rows(rows[:64])
    assert len(np.unique(words[:, :-1])) > 0.99 * words[:, :-1].size  # masks are not repeated
    mask_bits = np.unpackbits(eng.read_rows(rows[:2048])[:, :-1].view(np.uint8))
    assert abs(mask_bits.mean() - 0.5) < 0.002
    # determinism: a second engine with the same seed reproduces the stream; a different seed does not
    again = B200Engine(key, seed=9, eval_keys=eval_keys, device_encrypt=True)
    r2, o2 = again.encrypt_rows(bits[:64])
    assert np.array_equal(again.read_rows(r2), words)
    other = B200Engine(key, seed=10, eval_keys=eval_keys, device_encrypt=True)
    r3, o3 = other.encrypt_rows(bits[:64])
    assert not np.array_equal(other.read_rows(r3), words)
    # volume of config 5
    big = rng.integers(0, 2, size=2 * 4096 * 32)
    eng.synchronize()
    t0 = time.perf_counter()
    rows_big, owner_big = eng.encrypt_rows(big)
    eng.synchronize()
    dt = time.perf_counter() - t0
    assert np.array_equal(eng.decrypt_rows(rows_big), big)
    assert dt < 0.5, dt
    # the circuit layer runs on device-encrypted inputs unchanged
    assert decrypt_int(eng, add_bitwise(encrypt_int(eng, 1234, 12), encrypt_int(eng, 3000, 12))) == (1234 + 3000) % 4096
