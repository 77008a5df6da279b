"""Ring-side parameters and bootstrapping / key-switching key material.

The reference fixes only the LWE half of the parameter set (m = 500,
alpha = 2**-15, 32-bit torus, mu = 1/8: `encirc/torus.py:25-27,118-134`) and
replaces the bootstrap with a key-holding oracle (`encirc/engine.py:493-503`).
A real gate bootstrap needs the ring half as well.  We take the TFHE
"110-bit" gate-bootstrapping set the paper says its framework is analogous
to: N = 1024, k = 1, key switch t = 8 digits of base 2**2,
sigma_bk = 7.18e-9, sigma_ks = alpha -- with two changes that belong together:
the bootstrapping key is UNROLLED over pairs of LWE mask elements (Zhou et al.
2018, Bourse et al. 2018: three TRGSW samples s1, s2, s1*s2 per pair, half as
many CMux steps) and the gadget is l = 2 / Bg = 2**9 instead of 2**10, which
pays for the unrolling's larger key-noise term (3 external products per pair,
factors |X**a - 1|**2 ~ 2 and 4) so that the output noise stays where the
plain set had it.

Everything here runs once per engine on the host with numpy; the results are
raw torus words.  The device turns the bootstrapping key into its spectral
layout itself (`tfb_load_keys`, kernel K3 in `csrc/tfhe_b200.cu`).

Layouts (all int32 bit patterns of uint32 torus words):

  ring key   s'[N]                    bits 0/1
  bk         [ceil(n/2)][3][(k+1)*l][k+1][N]
                                      pair m, key j: TRGSW of s_2m (j = 0),
                                      s_2m+1 (j = 1), s_2m * s_2m+1 (j = 2; an
                                      odd n pads s_n = 0); row r = p*l + lvl is
                                      a TRLWE sample (a, b) of 0 under s' whose
                                      component p carries
                                      message * 2**(32 - (lvl+1)*bgbit)
  ksk        [N][t][n+1]              LWE_s( s'_i * 2**(32 - (j+1)*basebit) ),
                                      mask words then body

Random streams are `default_rng((seed, stream))` with streams 3 (ring key),
4 (bk) and 5 (ksk); the reference uses 0 (encrypt), 1 (oracle launches) and
2 (bench inputs) of the same seed (`encirc/engine.py:416-417`,
`encirc/bench.py:61`), so nothing collides.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .torus import SecretKey

RING_KEY_STREAM = 3
BK_STREAM = 4
KSK_STREAM = 5
BK_KEYS = 3  # TRGSW samples per pair of mask elements: s1, s2, s1 * s2


@dataclass(frozen=True)
class RingParams:
    """TRLWE / TRGSW / key-switch half of the parameter set."""

    N: int = 1024
    k: int = 1
    bk_l: int = 2
    bk_bgbit: int = 9
    ks_t: int = 8
    ks_basebit: int = 2
    bk_stdev: float = 7.18e-9
    ks_stdev: float | None = None  # None -> the LWE alpha

    def __post_init__(self) -> None:
        if self.k != 1:
            raise ValueError("only k = 1 is implemented")
        if self.N < 2 or self.N & (self.N - 1):
            raise ValueError("N must be a power of two")
        if self.bk_l * self.bk_bgbit > 32 or self.ks_t * self.ks_basebit > 31:
            raise ValueError("decomposition exceeds the 32-bit torus")

    @property
    def rows(self) -> int:
        """TRLWE rows per TRGSW sample: (k+1) * l."""
        return (self.k + 1) * self.bk_l


@dataclass(frozen=True, eq=False)
class EvaluationKeys:
    """Raw (coefficient-domain) evaluation keys plus the ring secret.

    The ring secret never leaves the host; it is kept so tests can audit
    intermediate ciphertexts (the extracted N-dimensional LWE sample)."""

    ring: RingParams
    n: int
    ring_key: np.ndarray  # int32[N]
    bk: np.ndarray  # int32[ceil(n/2)][3][rows][2][N]
    ksk: np.ndarray  # int32[N][t][n+1]


def negacyclic_mul_binary(a: np.ndarray, s: np.ndarray) -> np.ndarray:
    """a(X) * s(X) mod (X**N + 1, 2**32) for uint32 rows `a[..., N]` and a
    0/1 polynomial `s[N]`.

    Exact: a is split into 16-bit halves, each half goes through one float64
    matrix product against the signed circulant of s (entries in {-1,0,1});
    every partial sum stays below 2**26, far inside the 53-bit mantissa."""
    N = s.shape[0]
    j = np.arange(N)[:, None]
    m = np.arange(N)[None, :]
    circ = s[(m - j) % N].astype(np.float64) * np.where(m >= j, 1.0, -1.0)
    flat = a.reshape(-1, N).astype(np.uint32)
    lo = (flat & np.uint32(0xFFFF)).astype(np.float64) @ circ
    hi = (flat >> np.uint32(16)).astype(np.float64) @ circ
    out = lo.astype(np.int64) + (hi.astype(np.int64) << 16)
    return (out & 0xFFFFFFFF).astype(np.uint32).reshape(a.shape)


def _gauss_words(rng: np.random.Generator, stdev: float, size) -> np.ndarray:
    e = np.rint(rng.normal(0.0, stdev, size=size) * 4294967296.0).astype(np.int64)
    return (e & 0xFFFFFFFF).astype(np.uint32)


def generate_evaluation_keys(key: SecretKey, seed: int, ring: RingParams | None = None) -> EvaluationKeys:
    """Ring secret, bootstrapping key and key-switching key for `key`.

    A pure function of (key, seed, ring)."""
    ring = ring if ring is not None else RingParams()
    p = key.params
    if p.w != 32:
        raise ValueError("the B200 engine works on the 32-bit torus only")
    n, N, rows = p.m, ring.N, ring.rows
    s = key.bits.astype(np.uint32)

    ring_key = np.random.default_rng((seed, RING_KEY_STREAM)).integers(0, 2, size=N).astype(np.uint32)

    # bootstrapping key, unrolled over pairs of mask elements: 3 TRGSW samples per pair
    pairs = (n + 1) // 2
    s_pad = np.concatenate([s, np.zeros(2 * pairs - n, dtype=np.uint32)])
    s1, s2 = s_pad[0::2], s_pad[1::2]
    messages = np.stack([s1, s2, s1 * s2], axis=1)  # [pairs][3]
    rng = np.random.default_rng((seed, BK_STREAM))
    mask = rng.integers(0, 1 << 32, size=(pairs, BK_KEYS, rows, N), dtype=np.uint32)
    noise = _gauss_words(rng, ring.bk_stdev, (pairs, BK_KEYS, rows, N))
    body = negacyclic_mul_binary(mask, ring_key) + noise
    bk = np.stack([mask, body], axis=3)  # [pairs][3][rows][2][N]
    for p_idx in range(ring.k + 1):
        for lvl in range(ring.bk_l):
            gadget = np.uint32(1 << (32 - (lvl + 1) * ring.bk_bgbit))
            bk[:, :, p_idx * ring.bk_l + lvl, p_idx, 0] += messages * gadget

    # key-switching key: N * t LWE samples under s
    rng = np.random.default_rng((seed, KSK_STREAM))
    t = ring.ks_t
    ks_stdev = p.alpha if ring.ks_stdev is None else ring.ks_stdev
    ks_mask = rng.integers(0, 1 << 32, size=(N, t, n), dtype=np.uint32)
    ks_noise = _gauss_words(rng, ks_stdev, (N, t))
    weights = np.array([1 << (32 - (j + 1) * ring.ks_basebit) for j in range(t)], dtype=np.uint32)
    ks_body = ks_mask @ s + ks_noise + ring_key[:, None] * weights[None, :]
    ksk = np.concatenate([ks_mask, ks_body[..., None].astype(np.uint32)], axis=2)

    return EvaluationKeys(
        ring=ring,
        n=n,
        ring_key=ring_key.view(np.int32),
        bk=np.ascontiguousarray(bk).view(np.int32),
        ksk=np.ascontiguousarray(ksk).view(np.int32),
    )
