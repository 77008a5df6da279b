"""Integer / vector / matrix circuits on the cleartext engine: results against
native arithmetic, and launch / bootstrap counts against the counts the
reference itself produced (tests/golden/reference_meta.json)."""
import numpy as np
import pytest

from paper_2005_01945_b200 import (
    EncryptedInt, EncryptedIntVector, EncryptedMatrix, FlatLaunchTooLarge, GateKind, PoolConfig,
    ReferenceEngine, WorkerPool, accumulate_tree, add_bitwise, add_numberwise, as_signed, complement,
    decrypt_int, decrypt_matrix, decrypt_vector, encrypt_int, encrypt_matrix, encrypt_vector, mat_add,
    mat_mul_cannon, mat_mul_flat, mul_karatsuba, mul_naive, negate, shift_left, trivial_int, truncate,
    vec_add, vec_mul, zero_extend,
)

OPS = {"add_bitwise": add_bitwise, "add_numberwise": add_numberwise, "mul_naive": mul_naive,
       "mul_karatsuba": mul_karatsuba}


def wide_engine():
    return ReferenceEngine(pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 22)))


def check_scalar_circuits_against_reference(eng, golden, widths=(8, 16, 32)):
    for name, fn in OPS.items():
        for n in widths:
            rec = golden["meta"]["circuits"][f"{name}_{n}"]
            x, y = encrypt_int(eng, rec["a"], n), encrypt_int(eng, rec["b"], n)
            eng.reset_stats()
            r = fn(x, y)
            got = eng.stats.as_record()
            assert decrypt_int(eng, r) == rec["result"], (name, n)
            for field in ("single_gates", "compound_gates", "not_gates", "bootstraps", "batch_launches", "largest_batch"):
                assert got[field] == rec[field], (name, n, field)


def test_scalar_circuits_match_reference_counts(golden):
    check_scalar_circuits_against_reference(wide_engine(), golden)


def test_matrix_products_match_reference_counts(golden):
    eng = wide_engine()
    for name, fn in (("mat_mul_flat", mat_mul_flat), ("mat_mul_cannon", mat_mul_cannon)):
        for q in (2, 3, 4):
            rec = golden["meta"]["circuits"][f"{name}_{q}"]
            ea, eb = encrypt_matrix(eng, rec["A"], 16), encrypt_matrix(eng, rec["B"], 16)
            eng.reset_stats()
            c = fn(ea, eb)
            got = eng.stats.as_record()
            assert decrypt_matrix(eng, c) == rec["result"]
            for field in ("single_gates", "compound_gates", "bootstraps", "batch_launches", "largest_batch"):
                assert got[field] == rec[field], (name, q, field)


def test_adders_exhaustive_small(ref):
    n = 4
    for a in range(16):
        for b in range(0, 16, 3):
            x, y = encrypt_int(ref, a, n), encrypt_int(ref, b, n)
            assert decrypt_int(ref, add_bitwise(x, y)) == (a + b) % 16
            assert decrypt_int(ref, add_numberwise(x, y)) == (a + b) % 16
            assert decrypt_int(ref, mul_naive(x, y)) == a * b


def test_random_arithmetic(ref):
    rng = np.random.default_rng(7)
    for n in (5, 8, 12, 16):
        for _ in range(5):
            a, b = int(rng.integers(0, 1 << n)), int(rng.integers(0, 1 << n))
            x, y = encrypt_int(ref, a, n), encrypt_int(ref, b, n)
            assert decrypt_int(ref, add_bitwise(x, y)) == (a + b) % (1 << n)
            assert decrypt_int(ref, mul_naive(x, y)) == a * b
            assert decrypt_int(ref, mul_karatsuba(x, y)) == a * b
            assert decrypt_int(ref, negate(x)) == (-a) % (1 << n)
            assert decrypt_int(ref, complement(x)) == (~a) % (1 << n)


def test_gate_free_ops_and_errors(ref):
    x = encrypt_int(ref, 0b1011, 4)
    before = ref.snapshot_stats()
    assert decrypt_int(ref, shift_left(x, 2)) == 0b1100
    assert decrypt_int(ref, shift_left(x, 1, width=8)) == 0b10110
    assert decrypt_int(ref, shift_left(x, 9, width=6)) == 0
    assert decrypt_int(ref, zero_extend(x, 7)) == 0b1011
    assert decrypt_int(ref, truncate(x, 2)) == 0b11
    assert ref.snapshot_stats().delta(before).bootstraps == 0
    assert as_signed(0b1011, 4) == -5 and as_signed(5, 4) == 5
    assert decrypt_int(ref, encrypt_int(ref, -3, 4)) == 13
    assert decrypt_int(ref, trivial_int(ref, 9, 4)) == 9
    for bad in (lambda: shift_left(x, -1), lambda: zero_extend(x, 3), lambda: truncate(x, 0),
                lambda: truncate(x, 5), lambda: encrypt_int(ref, 16, 4), lambda: encrypt_int(ref, -9, 4),
                lambda: EncryptedInt(ref, []), lambda: add_bitwise(x, encrypt_int(ref, 1, 5)),
                lambda: add_bitwise(x, encrypt_int(ReferenceEngine(), 1, 4)), lambda: accumulate_tree([])):
        with pytest.raises(ValueError):
            bad()
    assert [b.engine is ref for b in x.bits] == [True] * 4 and x.width == 4


def test_lane_sharing_launch_counts():
    eng = wide_engine()
    for ell in (1, 4, 8, 16, 32):
        for n in (8, 16):
            u = encrypt_vector(eng, list(range(ell)), n)
            v = encrypt_vector(eng, list(range(ell, 2 * ell)), n)
            eng.reset_stats()
            w = vec_add(u, v)
            st = eng.stats
            assert (st.batch_launches, st.bootstraps, st.largest_batch) == (3 * n, 5 * n * ell, 2 * ell)
            assert decrypt_vector(eng, w) == [(2 * i + ell) % (1 << n) for i in range(ell)]
    u, v = encrypt_vector(eng, [3, 250, 17], 8), encrypt_vector(eng, [5, 250, 0], 8)
    eng.reset_stats()
    w = vec_mul(u, v)
    assert decrypt_vector(eng, w) == [15, 62500, 0]
    assert eng.stats.bootstraps == 3 * (11 * 64 - 80) and eng.stats.batch_launches == 1 + 3 * 6 * 8


def test_accumulate_tree_levels_and_value(ref):
    vals = [3, 5, 7, 11, 13, 200, 255]
    items = [encrypt_int(ref, v, 8) for v in vals]
    ref.reset_stats()
    total = accumulate_tree(items)
    assert decrypt_int(ref, total) == sum(vals) % 256
    assert ref.pool.level_counter() == 3
    assert ref.stats.batch_launches == 3 * 24  # every level shares one sliced addition


def test_matrix_shapes_and_guard():
    eng = wide_engine()
    a = encrypt_matrix(eng, [[1, 2, 3], [4, 5, 6]], 8)
    b = encrypt_matrix(eng, [[7, 8], [9, 10], [11, 12]], 8)
    assert decrypt_matrix(eng, mat_mul_flat(a, b)) == [[58, 64], [139, 154]]
    assert decrypt_matrix(eng, mat_add(a, a)) == [[2, 4, 6], [8, 10, 12]]
    with pytest.raises(ValueError):
        mat_mul_flat(a, a)
    with pytest.raises(ValueError):
        mat_mul_cannon(a, b)
    with pytest.raises(ValueError):
        mat_add(a, b)
    with pytest.raises(ValueError):
        encrypt_matrix(eng, [[1, 2], [3]], 8)
    with pytest.raises(IndexError):
        a.cell(2, 0)
    with pytest.raises(FlatLaunchTooLarge):
        mat_mul_flat(a, b, max_jobs=2 * 2 * 3 * 64)  # exactly the job count: refused
    mat_mul_flat(a, b, max_jobs=2 * 2 * 3 * 64 + 1)
    sq = encrypt_matrix(eng, [[1, 2], [3, 4]], 8)
    assert decrypt_matrix(eng, mat_mul_cannon(sq, sq)) == [[7, 10], [15, 22]]
    assert len(EncryptedIntVector(a.data)) == 6 and EncryptedMatrix(3, 2, a.data).cell(2, 1) is a.data[5]
