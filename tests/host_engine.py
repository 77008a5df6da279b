"""A host-memory LWE engine for CPU tests: the GateEngine contract with real
TFHE bootstraps evaluated by the C oracle.  TEST CODE (it calls oracle/); it
lets multi-process sharding logic and circuit plumbing run under gloo on a box
without a GPU.  Never used by the product path."""
import numpy as np

from oracle import tfhe_oracle as orc
from paper_2005_01945_b200.engine import IDENTITY_KIND_ID, GateEngine, _bit_value
from paper_2005_01945_b200.keys import generate_evaluation_keys
from paper_2005_01945_b200.torus import LweSample, gaussian_noise_words, uniform_words


class HostOracleEngine(GateEngine):
    name = "host-oracle-tfhe"

    def __init__(self, key, seed=0, pool=None, lazy=False):
        self._words = np.zeros((1024, key.params.m + 1), dtype=np.uint32)
        super().__init__(key.params, pool)
        self.lazy = bool(lazy)  # levelised execution (GateEngine._submit), as B200Engine runs by default
        self.key, self.seed = key, int(seed)
        self._enc_rng = np.random.default_rng((self.seed, 0))
        self.eval_keys = generate_evaluation_keys(key, self.seed)

    def _reserve_storage(self, rows):
        if rows > len(self._words):
            grown = np.zeros((max(rows, 2 * len(self._words)), self._words.shape[1]), dtype=np.uint32)
            grown[: len(self._words)] = self._words
            self._words = grown

    def _evaluate(self, kind_ids, x_rows, y_rows, out_rows):
        self._words[out_rows] = orc.gate_bootstrap_batch(
            self._words[x_rows], self._words[y_rows], np.asarray(kind_ids, np.uint8), self.params.mu.word,
            self.eval_keys.bk, self.eval_keys.ksk, fft=True)

    def _refresh(self, in_rows, out_rows):
        self._submit(np.full(len(in_rows), IDENTITY_KIND_ID, np.uint8), in_rows, in_rows, out_rows)

    def _negate_rows(self, rows):
        self._run_deferred()
        block = self._new_rows(len(rows))
        out = block.rows()
        self._words[out] = (0 - self._words[rows]).astype(np.uint32)
        self._bounds[out] = self._bounds[rows]
        return out, (block,)

    def _store_trivial(self, row, value):
        self._words[row] = 0
        self._words[row, -1] = self.params.message_word(value)

    def encrypt_rows(self, values):
        p = self.params
        block = self._new_rows(len(values))
        out = block.rows()
        for r, v in zip(out, values):
            a = uniform_words(p, self._enc_rng, p.m)
            e = int(gaussian_noise_words(p, self._enc_rng, 1)[0])
            self._words[r, :-1] = a
            self._words[r, -1] = (int(a @ self.key.bits) + p.message_word(_bit_value(v)) + e) & p.mask
        self._bounds[out] = self.fresh_bound
        return out, (block,)

    def decrypt_rows(self, rows):
        self._run_deferred()
        rows = np.asarray(rows, np.int64)
        self._check_decryptable(rows)
        w = self._words[rows]
        ph = w[:, -1] - w[:, :-1] @ self.key.bits.astype(np.uint32)
        return ((ph > 0) & (ph < np.uint32(self.params.half_word))).astype(np.int64)

    def read_rows(self, rows):
        self._run_deferred()
        return self._words[np.asarray(rows, np.int64)].copy()

    def write_rows(self, words, bounds):
        block = self._new_rows(len(words))
        out = block.rows()
        self._words[out] = words
        self._bounds[out] = bounds
        return out, (block,)

    def _adopt(self, sample, clear, bound):
        words = np.concatenate([np.asarray(sample.a, np.uint32), [np.uint32(sample.b)]])[None, :]
        rows, owners = self.write_rows(words, sample.noise_bound)
        return int(rows[0]), owners

    def _row_sample(self, row):
        self._run_deferred()
        w = self._words[row]
        return LweSample(w[:-1].copy(), int(w[-1]), float(self._bounds[row]), self.params.w)
