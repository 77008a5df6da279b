"""numpy restatement of the reference's CPU gate path (the `oracle-lwe` engine).

TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module.

This is the reference's own implementation of the hot path, restated
self-contained so it can travel to the GPU box (the reference under
/root/reference cannot): key generation (encirc/torus.py:226-230), fresh
encryption (encirc/torus.py:233-271), the integer linear combination
(encirc/torus.py:307-348), phase / decryption (encirc/torus.py:283-304) and the
batched launch of `OracleBootstrapEngine` (encirc/engine.py:458-514): gate
linear form, then a bootstrap that DECRYPTS with the secret key and
RE-ENCRYPTS under per-(launch, block) random streams.  It is pinned bit for
bit -- keys, ciphertext words, launch outputs, stats -- against golden vectors
produced by running the reference itself (tests/golden/make_golden.py).

The launch keeps the reference's cost structure on purpose (row stacking of
the inputs, one Python sample object per output), because bench.py times it
as the reference CPU baseline.
"""

from __future__ import annotations

import itertools

import numpy as np

M, ALPHA, W = 500, 2.0**-15, 32
MOD = 1 << W
MU = MOD // 8
HALF = MOD // 2
CLAMP = MU // 4  # fresh noise clipped to |e| <= CLAMP - 1
FRESH_BOUND = CLAMP / MOD
BLOCK = 256  # encirc/scheduler.py:22

# (cx, cy, offset/mu) in TWO_INPUT_KINDS order: AND OR NAND NOR XOR XNOR ANDNY ORNY
LINEAR = ((1, 1, -1), (1, 1, 1), (-1, -1, 1), (-1, -1, -1), (2, 2, 2), (-2, -2, -2), (-1, 1, -1), (-1, 1, 1))
TRUTH = ((0, 0, 0, 1), (0, 1, 1, 1), (1, 1, 1, 0), (1, 0, 0, 0), (0, 1, 1, 0), (1, 0, 0, 1), (0, 1, 0, 0), (1, 1, 0, 1))
MARGIN = (0.125, 0.125, 0.125, 0.125, 0.25, 0.25, 0.125, 0.125)


def keygen_bits(seed, m: int = M) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 2, size=m).astype(np.uint32)


def _noise_words(rng: np.random.Generator, size: int) -> np.ndarray:
    e = np.clip(np.rint(rng.normal(0.0, ALPHA, size=size) * float(MOD)), -(CLAMP - 1), CLAMP - 1)
    return (e.astype(np.int64) % MOD).astype(np.uint32)


class Sample:
    """(a, b, noise_bound): what the reference calls LweSample."""

    __slots__ = ("a", "b", "noise_bound")

    def __init__(self, a, b, noise_bound):
        self.a, self.b, self.noise_bound = a, int(b) % MOD, float(noise_bound)

    def words(self) -> np.ndarray:
        return np.concatenate([self.a, np.array([self.b], dtype=np.uint32)])


def encrypt(bits_key: np.ndarray, bit: int, rng: np.random.Generator) -> Sample:
    a = rng.integers(0, MOD, size=len(bits_key), dtype=np.uint32)
    e = int(_noise_words(rng, 1)[0])
    msg = MU if bit else MOD - MU
    return Sample(a, int(a @ bits_key) + msg + e, FRESH_BOUND)


def trivial(bit: int, m: int = M) -> Sample:
    return Sample(np.zeros(m, dtype=np.uint32), MU if bit else MOD - MU, 0.0)


def phase_word(bits_key: np.ndarray, c: Sample) -> int:
    return (c.b - int(c.a @ bits_key)) % MOD


def decrypt(bits_key: np.ndarray, c: Sample) -> int:
    if c.noise_bound >= (MU / MOD) / 2:
        raise ValueError("decryption unreliable")
    return 1 if 0 < phase_word(bits_key, c) < HALF else 0


def linear(samples, coeffs, offset_word: int = 0) -> Sample:
    a = np.zeros(len(samples[0].a), dtype=np.uint32)
    b, bound = offset_word, 0.0
    for c, k in zip(samples, coeffs):
        a = a + np.uint32(k % MOD) * c.a
        b += k * c.b
        bound += abs(k) * c.noise_bound
    return Sample(a, b, bound)


class OracleLweEngine:
    """Batched launches of the reference's oracle-LWE engine."""

    def __init__(self, bits_key: np.ndarray, seed: int = 0, max_batch: int = 4096):
        self.key = bits_key
        self.seed = int(seed)
        self.max_batch = int(max_batch)
        self._launch = itertools.count()
        self._enc_rng = np.random.default_rng((self.seed, 0))
        self.launches = 0
        self.bootstraps = 0
        self._cx = np.array([c[0] % MOD for c in LINEAR], dtype=np.uint32)
        self._cy = np.array([c[1] % MOD for c in LINEAR], dtype=np.uint32)
        self._off = np.array([(c[2] * MU) % MOD for c in LINEAR], dtype=np.uint64)
        self._ax = np.array([abs(c[0]) for c in LINEAR], dtype=np.float64)
        self._ay = np.array([abs(c[1]) for c in LINEAR], dtype=np.float64)
        self._margin = np.array(MARGIN)

    def encrypt(self, bit: int) -> Sample:
        return encrypt(self.key, bit, self._enc_rng)

    def decrypt(self, c: Sample) -> int:
        return decrypt(self.key, c)

    def launch(self, kind_ids, xs, ys) -> list:
        """One launch (encirc/engine.py:458-514)."""
        k = len(kind_ids)
        self.launches += 1
        self.bootstraps += k
        lid = next(self._launch)
        idx = np.asarray(kind_ids, dtype=np.intp)
        nbx = np.fromiter((c.noise_bound for c in xs), dtype=np.float64, count=k)
        nby = np.fromiter((c.noise_bound for c in ys), dtype=np.float64, count=k)
        if np.any(self._ax[idx] * nbx + self._ay[idx] * nby >= self._margin[idx]):
            raise ValueError("combined noise bound reaches the gate margin")
        ax = np.stack([c.a for c in xs])
        ay = np.stack([c.a for c in ys])
        bx = np.fromiter((c.b for c in xs), dtype=np.uint64, count=k)
        by = np.fromiter((c.b for c in ys), dtype=np.uint64, count=k)
        a_lin = self._cx[idx][:, None] * ax + self._cy[idx][:, None] * ay
        b_lin = ((self._cx[idx].astype(np.uint64) * bx + self._cy[idx].astype(np.uint64) * by + self._off[idx])
                 & np.uint64(MOD - 1)).astype(np.uint32)
        outs = []
        for blk in range(-(-k // BLOCK)):
            lo, hi = blk * BLOCK, min(k, (blk + 1) * BLOCK)
            rng = np.random.default_rng((self.seed, 1, lid, blk))
            ph = b_lin[lo:hi] - a_lin[lo:hi] @ self.key
            one = (ph > 0) & (ph < np.uint32(HALF))
            a_new = rng.integers(0, MOD, size=(hi - lo, len(self.key)), dtype=np.uint32)
            e = _noise_words(rng, hi - lo)
            b_new = a_new @ self.key + np.where(one, np.uint32(MU), np.uint32(MOD - MU)) + e
            for i in range(hi - lo):
                outs.append(Sample(a_new[i], int(b_new[i]), FRESH_BOUND))
        return outs

    def eval_gate_batch(self, kind_id: int, xs, ys) -> list:
        """Element-wise gate, split into launches of at most max_batch
        (encirc/engine.py:280-294 + encirc/scheduler.py:156-171)."""
        xs, ys = tuple(xs), tuple(ys)
        out = []
        for lo in range(0, len(xs), self.max_batch):
            hi = min(len(xs), lo + self.max_batch)
            out.extend(self.launch((kind_id,) * (hi - lo), xs[lo:hi], ys[lo:hi]))
        return out
