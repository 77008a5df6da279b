"""ctypes front-end of oracle/tfhe_gate_oracle.c (the exact CPU restatement of
TFHE gate bootstrapping).

TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may import this module.  Parity at the
ciphertext-coefficient level is UNPINNED by the reference (it has no
bootstrap: encirc/engine.py:493-503); see the header of the C file for what
is pinned and how.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtfhe_oracle.so")
RING_N = 1024

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile the C oracle next to its source (gcc, a second or two)."""
    src = os.path.join(_HERE, "tfhe_gate_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", _HERE, "CC=gcc", "libtfhe_oracle.so"], stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_gate_bootstrap_batch.argtypes = [
            _u32p, _u32p, _u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, _i32p, _i32p,
            ctypes.c_int, ctypes.c_int, _u32p, _u32p, _i32p,
        ]
        _lib.oracle_gate_bootstrap_batch.restype = None
        _lib.oracle_key_switch.argtypes = [_u32p, ctypes.c_int, _i32p, _u32p]
        _lib.oracle_key_switch.restype = None
        _lib.oracle_gate_linear.argtypes = [_u32p, _u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_int, _u32p]
        _lib.oracle_gate_linear.restype = None
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def gate_linear(x: np.ndarray, y: np.ndarray, kind: int, mu: int) -> np.ndarray:
    """cx*x + cy*y + off*mu on packed samples (n+1 words each)."""
    x = np.ascontiguousarray(x, dtype=np.uint32)
    y = np.ascontiguousarray(y, dtype=np.uint32)
    out = np.empty_like(x)
    lib().oracle_gate_linear(_ptr(x, _u32p), _ptr(y, _u32p), int(kind), int(mu), len(x) - 1, _ptr(out, _u32p))
    return out


def gate_bootstrap_batch(x, y, kinds, mu: int, bk: np.ndarray, ksk: np.ndarray, *, fft: bool = False,
                         threads: int = 0, want_ext: bool = False, want_bar: bool = False):
    """k bootstrapped gates on packed samples x, y [k][n+1].

    Returns out [k][n+1] (and, when asked, the extracted (N+1)-word samples
    before the key switch and the mod-switched words)."""
    x = np.ascontiguousarray(x, dtype=np.uint32)
    y = np.ascontiguousarray(y, dtype=np.uint32)
    kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
    k, n1 = x.shape
    n = n1 - 1
    bk = np.ascontiguousarray(bk, dtype=np.int32)
    ksk = np.ascontiguousarray(ksk, dtype=np.int32)
    assert bk.shape == ((n + 1) // 2, 3, 4, 2, RING_N) and ksk.shape == (RING_N, 8, n + 1)
    out = np.empty((k, n + 1), dtype=np.uint32)
    ext = np.empty((k, RING_N + 1), dtype=np.uint32) if want_ext else None
    bar = np.empty((k, n + 1), dtype=np.int32) if want_bar else None
    lib().oracle_gate_bootstrap_batch(
        _ptr(x, _u32p), _ptr(y, _u32p), _ptr(kinds, _u8p), k, n, int(mu), _ptr(bk, _i32p), _ptr(ksk, _i32p),
        int(bool(fft)), int(threads), _ptr(out, _u32p),
        _ptr(ext, _u32p) if want_ext else None, _ptr(bar, _i32p) if want_bar else None,
    )
    res = [out]
    if want_ext:
        res.append(ext)
    if want_bar:
        res.append(bar)
    return res[0] if len(res) == 1 else tuple(res)


def key_switch(ext: np.ndarray, ksk: np.ndarray) -> np.ndarray:
    ext = np.ascontiguousarray(ext, dtype=np.uint32)
    ksk = np.ascontiguousarray(ksk, dtype=np.int32)
    n = ksk.shape[2] - 1
    out = np.empty(n + 1, dtype=np.uint32)
    lib().oracle_key_switch(_ptr(ext, _u32p), n, _ptr(ksk, _i32p), _ptr(out, _u32p))
    return out


# ---- slow, independent numpy restatements used to cross-check the C code ------

def negacyclic_mul_numpy(d: np.ndarray, b: np.ndarray) -> np.ndarray:
    """d (*) b mod (X^N + 1, 2^32) with Python-int exact arithmetic via int64
    accumulation of 16-bit limbs (small N only needs seconds)."""
    N = len(d)
    d = d.astype(np.int64)
    b = b.astype(np.uint32).astype(np.int64)
    full = np.zeros(2 * N, dtype=object)
    for i in range(N):
        if d[i]:
            full[i : i + N] += int(d[i]) * b.astype(object)
    res = (full[:N] - full[N:]) % (1 << 32)
    return np.array(res, dtype=np.uint64).astype(np.uint32)


def ring_phase(acc_a: np.ndarray, acc_b: np.ndarray, ring_key: np.ndarray) -> np.ndarray:
    """b - a * s' for a TRLWE sample (used to audit bootstrapping-key rows)."""
    prod = negacyclic_mul_numpy(ring_key.astype(np.int64), acc_a)
    return (acc_b.astype(np.uint32) - prod).astype(np.uint32)


def lwe_phase(sample: np.ndarray, key_bits: np.ndarray) -> int:
    a = sample[:-1].astype(np.uint32)
    return int((int(sample[-1]) - int((a * key_bits.astype(np.uint32)).sum(dtype=np.uint64))) % (1 << 32))
