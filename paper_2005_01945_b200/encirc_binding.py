"""The B200 engine as a plug-in of the reference package itself (route B).

`bind(encirc)` takes the imported reference package and returns a class that subclasses the
reference's own `OracleBootstrapEngine` (`encirc/engine.py:405-514`) and overrides exactly the six
hooks of the boundary (`encirc/engine.py:322-340`: `trivial_bit`, `encrypt`, `decrypt`, `bootstrap`,
`_negate`, `execute_launch`).  Everything above it -- the reference's scheduler, adders, multipliers,
vector / matrix code, bench harness, CLI and its own test-suite -- then runs unchanged on the GPU:

    import encirc
    from paper_2005_01945_b200.encirc_binding import bind
    encirc.OracleBootstrapEngine = bind(encirc)        # or use the class directly

The reference's `EncBit.sample` is a plain attribute (`encirc/engine.py:134-157`), so device-resident
ciphertexts are represented by `DeviceSample`, a subclass of the reference's `LweSample` whose
`a` / `b` / `noise_bound` / `w` are read lazily from the device row.  Launches go to
`B200Engine.launch_rows`, i.e. they are counted, margin-checked and *recorded* at the call and
evaluated level by level when something reads a row; statistics are kept by the
reference's own `GateStats` on the outer engine.  Errors are re-raised as the reference's own types.

This module never imports `encirc` by itself: the product does not depend on the reference being
installed; whoever has the reference passes it in.
"""

from __future__ import annotations

import numpy as np

from . import engine as _eng
from . import torus as _torus
from .scheduler import PoolConfig, WorkerPool

_EVAL_KEY_CACHE: dict = {}


def _eval_keys_for(key, seed: int):
    """Evaluation keys are a pure function of (key, seed): share them between engines of one process
    (the reference's tests build a fresh engine per test)."""
    from .keys import generate_evaluation_keys

    tag = (key.bits.tobytes(), key.params.m, int(seed))
    if tag not in _EVAL_KEY_CACHE:
        if len(_EVAL_KEY_CACHE) >= 4:
            _EVAL_KEY_CACHE.pop(next(iter(_EVAL_KEY_CACHE)))
        _EVAL_KEY_CACHE[tag] = generate_evaluation_keys(key, seed)
    return _EVAL_KEY_CACHE[tag]


def bind(encirc, backend=None):
    """Build the engine class against the given reference package.

    backend: callable (key, seed) -> row engine with B200Engine's row API (`launch_rows`,
    `encrypt_rows`, `decrypt_rows`, `read_rows`, `write_rows`, `not_rows`, `trivial_bit`, `_refresh`);
    default: `B200Engine` on the current CUDA device.  (The CPU tests pass a host stand-in.)"""
    ref_engine, ref_torus = encirc.engine, encirc.torus
    RefBit, RefSample = ref_engine.EncBit, ref_torus.LweSample

    class DeviceSample(RefSample):
        """A ciphertext that lives in a device row; materialised on first attribute access."""

        __slots__ = ("_rows", "row", "_owner", "_cache")

        def __init__(self, rows_engine, row, owner):  # deliberately not calling LweSample.__init__
            self._rows, self.row, self._owner, self._cache = rows_engine, int(row), owner, None

        def _words(self):
            if self._cache is None:  # rows are write-once: a materialised copy never goes stale
                self._cache = self._rows.read_rows([self.row])[0]
            return self._cache

        a = property(lambda self: self._words()[:-1])
        b = property(lambda self: int(self._words()[-1]))
        noise_bound = property(lambda self: float(self._rows._bounds[self.row]))
        w = property(lambda self: self._rows.params.w)

    def _make_backend(key, seed):
        p = key.params
        mine = _torus.SecretKey(_torus.LweParams(m=p.m, alpha=p.alpha, w=p.w, mu=_torus.TorusElement(p.mu.word, p.w)),
                                np.asarray(key.bits).astype(_torus.word_dtype(p.w)))
        if backend is not None:
            return backend(mine, seed)
        pool = WorkerPool(PoolConfig(workers=1, max_batch=1 << 30))  # splitting is the reference scheduler's job
        return _eng.B200Engine(mine, seed=seed, pool=pool, eval_keys=_eval_keys_for(mine, seed))

    class B200BootstrapEngine(ref_engine.OracleBootstrapEngine):
        """Real TFHE gate bootstrapping on a B200 behind the reference's engine interface."""

        name = "b200-tfhe"

        def __init__(self, key, seed: int = 0, pool=None, **_ignored):
            super().__init__(key, seed, pool)  # tables (raises on a bad mu), stats, seed, pool
            self._rows = _make_backend(key, self.seed)

        # -- handles ----------------------------------------------------------------------------
        def _wrap(self, row, owner):
            return RefBit(self, sample=DeviceSample(self._rows, row, owner))

        def _row_of(self, bit, keep: list) -> int:
            s = bit.sample
            if type(s) is DeviceSample and s._rows is self._rows:
                return s.row
            # a host-side sample (hand-built by the caller, loaded from disk): adopt it with its bound
            words = np.concatenate([np.asarray(s.a, dtype=np.uint32), [np.uint32(s.b)]])[None, :]
            rows, owners = self._rows.write_rows(words, s.noise_bound)
            keep.append(owners)
            return int(rows[0])

        # -- the six hooks ----------------------------------------------------------------------
        def trivial_bit(self, value):
            inner = self._rows.trivial_bit(ref_engine._check_value(value))
            return self._wrap(inner.row, inner)

        def encrypt(self, value):
            rows, owners = self._rows.encrypt_rows([ref_engine._check_value(value)])
            return self._wrap(rows[0], owners)

        def decrypt(self, bit) -> int:
            self._check_bit(bit)
            keep: list = []
            try:
                return int(self._rows.decrypt_rows(np.array([self._row_of(bit, keep)], np.int64))[0])
            except _torus.DecryptionUnreliableError as exc:
                raise ref_torus.DecryptionUnreliableError(str(exc)) from None

        def bootstrap(self, bit):
            self._check_bit(bit)
            mu = self.params.mu_float
            if bit.sample.noise_bound >= mu:
                raise ref_engine.BootstrapMarginError(f"noise_bound {bit.sample.noise_bound:.3g} >= margin {mu:.3g}")
            self._count_launch(1)
            keep: list = []
            out = self._rows.bootstrap(_eng.EncBit(self._rows, _row=self._row_of(bit, keep), _owner=keep))
            return self._wrap(out.row, out)

        def _negate(self, x):
            keep: list = []
            rows, owners = self._rows.not_rows(np.array([self._row_of(x, keep)], np.int64))
            return self._wrap(rows[0], owners)

        def execute_launch(self, kinds, xs, ys, pool) -> list:
            k = len(kinds)
            self._count_launch(k)
            ids = np.fromiter((self._kind_index[kd] for kd in kinds), dtype=np.uint8, count=k)
            keep: list = []
            x_rows = np.fromiter((self._row_of(b, keep) for b in xs), dtype=np.int64, count=k)
            y_rows = np.fromiter((self._row_of(b, keep) for b in ys), dtype=np.int64, count=k)
            try:
                rows, owners = self._rows.launch_rows(ids, x_rows, y_rows)
            except _eng.BootstrapMarginError as exc:
                raise ref_engine.BootstrapMarginError(str(exc)) from None
            return [self._wrap(r, owners) for r in rows]

        def synchronize(self) -> None:
            self._rows.synchronize()

    B200BootstrapEngine.DeviceSample = DeviceSample
    return B200BootstrapEngine
