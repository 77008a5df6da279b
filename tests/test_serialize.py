"""Wire formats against bytes produced by the reference's serialize.py, and the
strictness of the loaders (reference pkg/tests/test_serialize.py:95-118)."""
import numpy as np
import pytest

from paper_2005_01945_b200 import (
    LweParams, LweSample, ReferenceEngine, decrypt_int, decrypt_matrix, decrypt_vector, encrypt_int,
    encrypt_matrix, encrypt_vector, generate_evaluation_keys, keygen,
)
from paper_2005_01945_b200.serialize import (
    FormatError, dump_eval_keys, dump_int, dump_key, dump_matrix, dump_params, dump_sample, dump_vector,
    load_eval_keys, load_int, load_key, load_key_file, load_matrix, load_params, load_sample, load_vector,
    save_key,
)
from tests.host_engine import HostOracleEngine


@pytest.fixture
def host_engine(key, eval_keys):
    eng = HostOracleEngine.__new__(HostOracleEngine)
    # reuse the session evaluation keys instead of regenerating them
    eng._words = np.zeros((1024, key.params.m + 1), dtype=np.uint32)
    from paper_2005_01945_b200.engine import GateEngine

    GateEngine.__init__(eng, key.params, None)
    eng.key, eng.seed = key, 9
    eng._enc_rng = np.random.default_rng((9, 0))
    eng.eval_keys = eval_keys
    return eng


def test_params_key_sample_bytes_match_reference(golden, params, key):
    assert dump_params(params) == golden["ser_params"].tobytes()
    assert dump_key(key) == golden["ser_key11"].tobytes()
    w = golden["enc5_words"][0]
    s = LweSample(w[:-1], int(w[-1]), params.fresh_noise_bound, 32)
    assert dump_sample(s) == golden["ser_sample"].tobytes()
    back = load_sample(golden["ser_sample"].tobytes())
    assert np.array_equal(back.a, w[:-1]) and back.b == int(w[-1]) and back.noise_bound == 2.0**-5 and back.w == 32
    assert load_params(golden["ser_params"].tobytes()) == params
    k2 = load_key(golden["ser_key11"].tobytes())
    assert np.array_equal(k2.bits, key.bits) and k2.params == params


def test_ciphertext_containers_match_reference_bytes(golden, host_engine):
    x = encrypt_int(host_engine, 11, 4)
    vec = encrypt_vector(host_engine, [3, 5], 3)
    mat = encrypt_matrix(host_engine, [[1, 2], [3, 0]], 2)
    assert dump_int(x) == golden["ser_int"].tobytes()
    assert dump_vector(vec) == golden["ser_vector"].tobytes()
    assert dump_matrix(mat) == golden["ser_matrix"].tobytes()
    assert decrypt_int(host_engine, load_int(golden["ser_int"].tobytes(), host_engine)) == 11
    assert decrypt_vector(host_engine, load_vector(golden["ser_vector"].tobytes(), host_engine)) == [3, 5]
    assert decrypt_matrix(host_engine, load_matrix(golden["ser_matrix"].tobytes(), host_engine)) == [[1, 2], [3, 0]]
    assert load_int(dump_int(x), host_engine).bits[0].noise_bound == host_engine.fresh_bound


def test_loaders_are_strict(golden, host_engine, tmp_path, key):
    blob = golden["ser_int"].tobytes()
    for bad in (b"ENC\x02" + blob[4:], blob[:4] + b"V" + blob[5:], blob[:-1], blob + b"\x00"):
        with pytest.raises(FormatError):
            load_int(bad, host_engine)
    with pytest.raises(FormatError):
        load_sample(golden["ser_params"].tobytes())
    other = HostOracleEngine.__new__(HostOracleEngine)
    from paper_2005_01945_b200.engine import GateEngine

    small = keygen(LweParams(m=8), seed=1)
    other._words = np.zeros((16, 9), dtype=np.uint32)
    GateEngine.__init__(other, small.params, None)
    with pytest.raises(FormatError):
        load_int(blob, other)  # dimensions do not match the engine
    kb = bytearray(golden["ser_key11"].tobytes())
    kb[-1] = 2
    with pytest.raises(FormatError):
        load_key(bytes(kb))
    with pytest.raises(ValueError):
        dump_int(encrypt_int(ReferenceEngine(), 3, 4))  # cleartext integers have no wire form
    path = tmp_path / "k.bin"
    save_key(str(path), key)
    assert np.array_equal(load_key_file(str(path)).bits, key.bits)


def test_evaluation_keys_roundtrip(eval_keys):
    blob = dump_eval_keys(eval_keys)
    back = load_eval_keys(blob)
    assert back.n == eval_keys.n and back.ring == eval_keys.ring
    assert np.array_equal(back.bk, eval_keys.bk) and np.array_equal(back.ksk, eval_keys.ksk)
    assert np.array_equal(back.ring_key, eval_keys.ring_key)
    with pytest.raises(FormatError):
        load_eval_keys(blob[:-4])


def test_untrusted_sample_header_cannot_size_an_allocation():
    """A sample payload announcing a huge m must fail as a truncated payload (FormatError), not while numpy
    builds a record type from the header (reference contract: encirc/serialize.py:46-58)."""
    import struct

    for m in (0xFFFFFFFF, 0x10000000, 501):
        blob = b"ENC\x01S" + struct.pack("<BI", 32, m) + b"\x00" * 64
        with pytest.raises(FormatError):
            load_sample(blob)
