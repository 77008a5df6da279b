"""Wire formats for parameters, keys and ciphertexts.

Byte-compatible with the reference's `encirc/serialize.py` (checked against
bytes the reference itself produced, tests/golden): 4-byte magic b"ENC\\x01",
one kind byte, little-endian fields, torus words always 8 bytes wide,
length-prefixed sequences:

    params  'P'  u32 m | u8 w | f64 alpha | u64 mu_word
    key     'K'  params body | u32 count | count key bits, one byte each
    sample  'S'  u8 w | u32 m | m x u64 mask words | u64 body | f64 bound
    int     'I'  u32 width | width sample bodies
    vector  'V'  u32 length | length int bodies
    matrix  'M'  u32 rows | u32 cols | rows*cols int bodies, row-major
    evalkey 'E'  (extension) u32 n | u32 N | u8 l | u8 bgbit | u8 t | u8 basebit |
                 N ring-key bytes | bk int32[ceil(n/2)][3][2l][2][N] | ksk int32[N][t][n+1]

Ciphertexts of a device engine are moved in bulk: all sample bodies of an
integer / vector / matrix are one structured numpy array filled from one
`read_rows` (device -> host) and adopted by one `write_rows`.  Loading is as
strict as the reference's: bad magic, wrong kind, truncation, trailing bytes,
out-of-range words and dimension mismatches raise `FormatError`.
"""

from __future__ import annotations

import struct

import numpy as np

from .integers import EncryptedInt
from .keys import BK_KEYS, EvaluationKeys, RingParams
from .linalg import EncryptedIntVector, EncryptedMatrix
from .torus import LweParams, LweSample, SecretKey, TorusElement, word_dtype

MAGIC = b"ENC\x01"


class FormatError(ValueError):
    """Malformed or wrong-kind serialized payload."""


class _Cursor:
    def __init__(self, data: bytes, kind: bytes):
        self.view = memoryview(bytes(data))
        self.at = 0
        magic = bytes(self.take(4))
        if magic != MAGIC:
            raise FormatError(f"bad magic/version {magic!r}, expected {MAGIC!r}")
        got = bytes(self.take(1))
        if got != kind:
            raise FormatError(f"payload kind {got!r}, expected {kind!r}")

    def take(self, size: int):
        if size < 0 or self.at + size > len(self.view):
            raise FormatError("truncated payload")
        chunk = self.view[self.at : self.at + size]
        self.at += size
        return chunk

    def fields(self, fmt: str):
        return struct.unpack("<" + fmt, self.take(struct.calcsize("<" + fmt)))

    def finish(self) -> None:
        if self.at != len(self.view):
            raise FormatError(f"{len(self.view) - self.at} trailing bytes")


# -- params / secret key ------------------------------------------------------------------


def _pack_params(p: LweParams) -> bytes:
    return struct.pack("<IBdQ", p.m, p.w, p.alpha, p.mu.word)


def _unpack_params(c: _Cursor) -> LweParams:
    m, w, alpha, mu_word = c.fields("IBdQ")
    try:
        return LweParams(m=m, alpha=alpha, w=w, mu=TorusElement(mu_word, w))
    except ValueError as exc:
        raise FormatError(f"invalid parameters: {exc}") from exc


def dump_params(params: LweParams) -> bytes:
    return MAGIC + b"P" + _pack_params(params)


def load_params(data: bytes) -> LweParams:
    c = _Cursor(data, b"P")
    params = _unpack_params(c)
    c.finish()
    return params


def dump_key(key: SecretKey) -> bytes:
    bits = np.asarray(key.bits, dtype=np.uint8).tobytes()
    return MAGIC + b"K" + _pack_params(key.params) + struct.pack("<I", len(bits)) + bits


def load_key(data: bytes) -> SecretKey:
    c = _Cursor(data, b"K")
    params = _unpack_params(c)
    (count,) = c.fields("I")
    if count != params.m:
        raise FormatError(f"key length {count} does not match m={params.m}")
    bits = np.frombuffer(c.take(count), dtype=np.uint8)
    if bits.size and bits.max() > 1:
        raise FormatError("key bits must be 0 or 1")
    c.finish()
    return SecretKey(params, bits.astype(params.dtype))


def save_key(path: str, key: SecretKey) -> None:
    with open(path, "wb") as fh:
        fh.write(dump_key(key))


def load_key_file(path: str) -> SecretKey:
    with open(path, "rb") as fh:
        return load_key(fh.read())


# -- samples ---------------------------------------------------------------------------------


def _record_dtype(m: int) -> np.dtype:
    """One serialized sample body as a packed record."""
    return np.dtype([("w", "u1"), ("m", "<u4"), ("a", "<u8", (m,)), ("b", "<u8"), ("bound", "<f8")])


def _records(words: np.ndarray, bounds: np.ndarray, w: int) -> bytes:
    """Packed sample bodies for ciphertext words [k][m+1] and their bounds."""
    k, m1 = words.shape
    rec = np.empty(k, dtype=_record_dtype(m1 - 1))
    rec["w"], rec["m"] = w, m1 - 1
    rec["a"] = words[:, :-1]
    rec["b"] = words[:, -1]
    rec["bound"] = bounds
    return rec.tobytes()


def _take_records(c: _Cursor, count: int, params: LweParams | None):
    """`count` sample bodies -> (words [count][m+1], bounds, w).  With `params`
    every record must match the engine's dimensions."""
    if count == 0:
        raise FormatError("empty sample sequence")
    head = bytes(c.view[c.at : c.at + 5])
    if len(head) < 5:
        raise FormatError("truncated payload")
    w, m = struct.unpack("<BI", head)
    if not 1 <= w <= 64:
        raise FormatError(f"bad torus precision {w}")
    if params is not None and (w != params.w or m != params.m):
        raise FormatError("sample dimensions do not match the engine parameters")
    need = (8 * m + 21) * count  # u8 w, u32 m, m x u64 mask, u64 body, f64 bound per record
    if need > len(c.view) - c.at:  # before the dtype exists: m comes from an untrusted header
        raise FormatError("truncated payload")
    dt = _record_dtype(m)
    rec = np.frombuffer(c.take(need), dtype=dt)
    if np.any(rec["w"] != w) or np.any(rec["m"] != m):
        raise FormatError("sample dimensions do not match the engine parameters" if params is not None
                          else "mixed sample dimensions")
    limit = (1 << w) - 1
    if m and int(rec["a"].max()) > limit:
        raise FormatError("mask word exceeds torus modulus")
    words = np.empty((count, m + 1), dtype=word_dtype(w))
    words[:, :-1] = rec["a"]
    words[:, -1] = rec["b"] & np.uint64(limit)  # the reference reduces the body word too (LweSample masks b)
    return words, rec["bound"].copy(), w


def dump_sample(sample: LweSample) -> bytes:
    words = np.concatenate([np.asarray(sample.a, dtype=np.uint64), [np.uint64(sample.b)]])[None, :]
    return MAGIC + b"S" + _records(words, np.array([sample.noise_bound]), sample.w)


def load_sample(data: bytes) -> LweSample:
    c = _Cursor(data, b"S")
    words, bounds, w = _take_records(c, 1, None)
    c.finish()
    return LweSample(words[0, :-1].copy(), int(words[0, -1]), float(bounds[0]), w)


# -- encrypted integers / vectors / matrices -------------------------------------------------------


def _engine_words(engine, rows: np.ndarray):
    if not hasattr(engine, "read_rows"):
        raise ValueError("only LWE-backed integers can be serialized")
    return engine.read_rows(rows), engine._bounds[rows]


def _ints_body(items) -> bytes:
    """Concatenated int bodies of same-engine integers, one bulk read."""
    engine = items[0].engine
    rows = np.concatenate([v._rows for v in items])
    words, bounds = _engine_words(engine, rows)
    w = engine.params.w
    out, pos = [], 0
    for v in items:
        out.append(struct.pack("<I", v.width))
        out.append(_records(words[pos : pos + v.width], bounds[pos : pos + v.width], w))
        pos += v.width
    return b"".join(out)


def _take_ints(c: _Cursor, count: int, engine) -> list:
    if not hasattr(engine, "write_rows"):
        raise ValueError("only LWE engines can load ciphertexts")
    parts, widths = [], []
    for _ in range(count):
        (width,) = c.fields("I")
        if width < 1:
            raise FormatError("integer width must be >= 1")
        words, bounds, _ = _take_records(c, width, engine.params)
        parts.append((words, bounds))
        widths.append(width)
    rows, owners = engine.write_rows(np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))
    out, pos = [], 0
    for width in widths:
        out.append(EncryptedInt._wrap(engine, rows[pos : pos + width], owners))
        pos += width
    return out


def dump_int(x: EncryptedInt) -> bytes:
    return MAGIC + b"I" + _ints_body([x])


def load_int(data: bytes, engine) -> EncryptedInt:
    c = _Cursor(data, b"I")
    (x,) = _take_ints(c, 1, engine)
    c.finish()
    return x


def dump_vector(vec: EncryptedIntVector) -> bytes:
    return MAGIC + b"V" + struct.pack("<I", len(vec)) + _ints_body(list(vec.items))


def load_vector(data: bytes, engine) -> EncryptedIntVector:
    c = _Cursor(data, b"V")
    (length,) = c.fields("I")
    if length < 1:
        raise FormatError("vector needs at least one element")
    items = _take_ints(c, length, engine)
    c.finish()
    return EncryptedIntVector(items)


def dump_matrix(mat: EncryptedMatrix) -> bytes:
    return MAGIC + b"M" + struct.pack("<II", mat.rows, mat.cols) + _ints_body(list(mat.data))


def load_matrix(data: bytes, engine) -> EncryptedMatrix:
    c = _Cursor(data, b"M")
    rows, cols = c.fields("II")
    if rows < 1 or cols < 1:
        raise FormatError("matrix shape must be at least 1x1")
    items = _take_ints(c, rows * cols, engine)
    c.finish()
    return EncryptedMatrix(rows, cols, items)


# -- evaluation keys (extension; the reference has none) ---------------------------------------------


def dump_eval_keys(keys: EvaluationKeys) -> bytes:
    r = keys.ring
    head = struct.pack("<IIBBBB", keys.n, r.N, r.bk_l, r.bk_bgbit, r.ks_t, r.ks_basebit)
    return b"".join([MAGIC, b"E", head, np.asarray(keys.ring_key, dtype=np.uint8).tobytes(),
                     np.ascontiguousarray(keys.bk, dtype="<i4").tobytes(),
                     np.ascontiguousarray(keys.ksk, dtype="<i4").tobytes()])


def load_eval_keys(data: bytes) -> EvaluationKeys:
    c = _Cursor(data, b"E")
    n, N, l, bgbit, t, basebit = c.fields("IIBBBB")
    try:
        ring = RingParams(N=N, bk_l=l, bk_bgbit=bgbit, ks_t=t, ks_basebit=basebit)
    except ValueError as exc:
        raise FormatError(f"invalid ring parameters: {exc}") from exc
    if n < 1:
        raise FormatError("LWE dimension must be >= 1")
    ring_key = np.frombuffer(c.take(N), dtype=np.uint8)
    if ring_key.max(initial=0) > 1:
        raise FormatError("ring key bits must be 0 or 1")
    pairs = (n + 1) // 2  # the bootstrapping key is unrolled over pairs of mask elements: keys s1, s2, s1*s2
    bk = np.frombuffer(c.take(4 * pairs * BK_KEYS * ring.rows * 2 * N), dtype="<i4").reshape(pairs, BK_KEYS, ring.rows, 2, N)
    ksk = np.frombuffer(c.take(4 * N * t * (n + 1)), dtype="<i4").reshape(N, t, n + 1)
    c.finish()
    return EvaluationKeys(ring=ring, n=n, ring_key=ring_key.astype(np.int32), bk=bk.copy(), ksk=ksk.copy())
