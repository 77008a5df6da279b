"""Gate engines: the hot-path boundary.

Mirror of the reference's L2 layer (`encirc/engine.py`): `GateKind`,
`GateStats`, `EncBit`, `GateEngine`, `ReferenceEngine`, `BootstrapMarginError`,
`truth_table`, `TWO_INPUT_KINDS`, with the same call signatures, counters and
error behaviour.  The reference's third engine, `OracleBootstrapEngine`
(`encirc/engine.py:405-514`), bootstraps by decrypting with the secret key and
re-encrypting; `B200Engine` takes its place and performs real TFHE gate
bootstrapping on the GPU through the C ABI in include/tfhe_b200.h.

Design difference from the reference: ciphertexts live in a row pool (device
memory for `B200Engine`, a numpy array for the cleartext `ReferenceEngine`)
and an `EncBit` is a (engine, row) handle.  All evaluation entry points have
an index-array form (`gate_rows`, `compound_rows`, `not_rows`, ...) that the
circuit layer uses, so a launch of 2**16 gates costs a handful of numpy calls
and one kernel sequence instead of 2**16 Python objects.  The handle-level API
of the reference (`eval_gate`, `eval_gate_batch`, `eval_compound_batch`,
`execute_launch(kinds, xs, ys, pool)`, ...) is kept on top of it.
"""

from __future__ import annotations

import bisect
import os
import enum
import itertools
from dataclasses import dataclass, fields, replace

import numpy as np

from .scheduler import JobBatch, WorkerPool
from .torus import (
    DecryptionUnreliableError,
    LweParams,
    LweSample,
    SecretKey,
    gaussian_noise_words,
    uniform_words,
)


class BootstrapMarginError(Exception):
    """Combined input noise bound reaches the gate's decision margin."""


class GateKind(enum.Enum):
    """ANDNY = (not x) and y; ORNY = (not x) or y; NOT is bootstrap-free."""

    AND = "AND"
    OR = "OR"
    XOR = "XOR"
    NAND = "NAND"
    NOR = "NOR"
    XNOR = "XNOR"
    ANDNY = "ANDNY"
    ORNY = "ORNY"
    NOT = "NOT"


# kind -> (truth table indexed by (x << 1) | y, (cx, cy, offset in units of mu)).
# The linear forms are the reference's (`encirc/engine.py:77-86`), which are the
# TFHE library's gate table; dict order fixes the kind ids used on the device.
_GATES = {
    GateKind.AND: ((0, 0, 0, 1), (1, 1, -1)),
    GateKind.OR: ((0, 1, 1, 1), (1, 1, 1)),
    GateKind.NAND: ((1, 1, 1, 0), (-1, -1, 1)),
    GateKind.NOR: ((1, 0, 0, 0), (-1, -1, -1)),
    GateKind.XOR: ((0, 1, 1, 0), (2, 2, 2)),
    GateKind.XNOR: ((1, 0, 0, 1), (-2, -2, -2)),
    GateKind.ANDNY: ((0, 1, 0, 0), (-1, 1, -1)),
    GateKind.ORNY: ((1, 1, 0, 1), (-1, 1, 1)),
}
TWO_INPUT_KINDS = tuple(_GATES)
KIND_ID = {kind: i for i, kind in enumerate(TWO_INPUT_KINDS)}
IDENTITY_KIND_ID = len(TWO_INPUT_KINDS)  # device-side "refresh x alone"


def truth_table(kind: GateKind) -> tuple:
    if kind is GateKind.NOT:
        return (1, 0)
    return _GATES[kind][0]


@dataclass
class GateStats:
    """Cumulative counters; `largest_batch` is a high-water mark."""

    single_gates: int = 0
    compound_gates: int = 0
    not_gates: int = 0
    bootstraps: int = 0
    batch_launches: int = 0
    largest_batch: int = 0

    def snapshot(self) -> "GateStats":
        return replace(self)

    def reset(self) -> None:
        for f in fields(self):
            setattr(self, f.name, 0)

    def delta(self, earlier: "GateStats") -> "GateStats":
        diff = {f.name: getattr(self, f.name) - getattr(earlier, f.name) for f in fields(self)}
        diff["largest_batch"] = self.largest_batch
        return GateStats(**diff)

    def as_record(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}


# -- row storage -----------------------------------------------------------------


class RowBlock:
    """Owner of the pool rows [start, start + count); returns them to the
    allocator when the last handle or integer referring to it is dropped."""

    __slots__ = ("_alloc", "start", "count", "__weakref__")

    def __init__(self, alloc: "RowAllocator", start: int, count: int):
        self._alloc, self.start, self.count = alloc, start, count

    def rows(self) -> np.ndarray:
        return np.arange(self.start, self.start + self.count, dtype=np.int64)

    def __del__(self):
        alloc = self._alloc
        if alloc is not None:
            alloc._release(self.start, self.count)


class RowAllocator:
    """First-fit extent allocator over an unbounded row index space."""

    def __init__(self) -> None:
        self._free_starts: list[int] = []
        self._free_counts: list[int] = []
        self.top = 0  # rows >= top have never been handed out (or were given back)
        self.hold = False  # while launches are deferred, freed rows wait in quarantine (they may still be read)
        self._held: list[tuple[int, int]] = []

    def alloc(self, count: int) -> RowBlock:
        for i, c in enumerate(self._free_counts):
            if c >= count:
                start = self._free_starts[i]
                if c == count:
                    del self._free_starts[i], self._free_counts[i]
                else:
                    self._free_starts[i] += count
                    self._free_counts[i] -= count
                return RowBlock(self, start, count)
        start = self.top
        self.top += count
        return RowBlock(self, start, count)

    def end_hold(self) -> None:
        self.hold = False
        held, self._held = self._held, []
        for start, count in held:
            self._release(start, count)

    def _release(self, start: int, count: int) -> None:
        if self.hold:
            self._held.append((start, count))
            return
        starts, counts = self._free_starts, self._free_counts
        i = bisect.bisect_left(starts, start)
        starts.insert(i, start)
        counts.insert(i, count)
        if i + 1 < len(starts) and starts[i] + counts[i] == starts[i + 1]:
            counts[i] += counts[i + 1]
            del starts[i + 1], counts[i + 1]
        if i > 0 and starts[i - 1] + counts[i - 1] == starts[i]:
            counts[i - 1] += counts[i]
            del starts[i], counts[i]
            i -= 1
        if starts[i] + counts[i] == self.top:
            self.top = starts[i]
            del starts[i], counts[i]


class EncBit:
    """Handle to one encrypted bit: the owning engine and a pool row.

    `EncBit(engine, sample=...)` / `EncBit(engine, clear=..., bound=...)` adopt
    an explicit sample or cleartext value, as the reference's constructor does
    (`encirc/engine.py:143-147`); engines create handles with `_row=`.
    """

    __slots__ = ("engine", "row", "_owner")

    def __init__(self, engine, sample: LweSample | None = None, clear: int | None = None,
                 bound: float | None = None, *, _row: int | None = None, _owner=None):
        self.engine = engine
        if _row is None:
            _row, _owner = engine._adopt(sample, clear, bound)
        self.row = int(_row)
        self._owner = _owner

    @property
    def noise_bound(self) -> float:
        return float(self.engine._bounds[self.row])

    @property
    def sample(self) -> LweSample | None:
        return self.engine._row_sample(self.row)

    @property
    def clear(self) -> int | None:
        return self.engine._row_clear(self.row)

    def __repr__(self) -> str:
        tag = "lwe" if self.engine._row_clear(self.row) is None else f"clear={self.clear}"
        return f"EncBit({tag}, noise_bound={self.noise_bound:.3g})"


def _bit_value(value) -> int:
    if value not in (0, 1):
        raise ValueError(f"bit value must be 0 or 1, got {value!r}")
    return int(value)


class GateEngine:
    """Gate semantics shared by every engine: tables, margins, stats, dispatch."""

    name = "abstract"

    def __init__(self, params: LweParams, pool: WorkerPool | None = None):
        self.params = params
        self.pool = pool if pool is not None else WorkerPool()
        self.stats = GateStats()
        self._alloc = RowAllocator()
        self._bounds = np.zeros(1024, dtype=np.float64)
        self._build_tables()
        self._trivial: dict[int, EncBit] = {}
        self._deferred: dict = {}          # level -> launches counted but not yet executed (lazy engines only)
        self._deferred_gates = 0
        self._deferred_launches = 0
        self._depth_done = 0               # highest level of the current queue epoch already handed to the device
        self._row_level = np.zeros(1024, dtype=np.int32)  # level of the queued launch that will write a row (0: none)
        self.physical_launches = 0         # _evaluate calls (logical launches are stats.batch_launches)

    # -- tables ----------------------------------------------------------------------
    def _build_tables(self) -> None:
        """Check every linear form against its truth table at this mu and
        derive the decision margins (reference `encirc/engine.py:179-224`)."""
        p = self.params
        mod, half, mu = p.modulus, p.half_word, p.mu.word
        msg = np.array([mod - mu, mu], dtype=object)  # encodings of 0 and 1
        self._kind_index = dict(KIND_ID)
        coeffs = np.array([_GATES[k][1] for k in TWO_INPUT_KINDS], dtype=np.int64)
        margins = []
        for kind, (cx, cy, off) in zip(TWO_INPUT_KINDS, coeffs.tolist()):
            truth = _GATES[kind][0]
            worst = None
            for idx in range(4):
                target = (cx * msg[idx >> 1] + cy * msg[idx & 1] + off * mu) % mod
                if (1 if 0 < target < half else 0) != truth[idx]:
                    raise ValueError(f"mu={p.mu!r} breaks the {kind.value} linearization")
                gap = min(target, mod - target, abs(target - half))
                worst = gap if worst is None else min(worst, gap)
            if worst <= 0:
                raise ValueError(f"mu={p.mu!r} leaves no decision margin for {kind.value}")
            margins.append(worst / mod)
        self._coeffs = coeffs
        self._absx = np.abs(coeffs[:, 0]).astype(np.float64)
        self._absy = np.abs(coeffs[:, 1]).astype(np.float64)
        self._margins = np.array(margins)
        self._safe_bound = float(np.min(self._margins / (self._absx + self._absy)))
        self._truth = np.array([_GATES[k][0] for k in TWO_INPUT_KINDS], dtype=np.uint8)

    def gate_margin(self, kind: GateKind) -> float:
        return float(self._margins[self._kind_index[kind]])

    # -- bookkeeping -------------------------------------------------------------------
    @property
    def fresh_bound(self) -> float:
        return self.params.fresh_noise_bound

    def reset_stats(self) -> None:
        self.stats.reset()

    def snapshot_stats(self) -> GateStats:
        return self.stats.snapshot()

    def _check_bit(self, b) -> None:
        if not isinstance(b, EncBit) or b.engine is not self:
            raise ValueError("input bit does not belong to this engine")

    def _check_two_input(self, kind: GateKind) -> None:
        if kind not in _GATES:
            raise ValueError(f"{kind!r} is not a two-input gate kind")

    def _count_launch(self, k: int) -> None:
        st = self.stats
        st.batch_launches += 1
        st.bootstraps += k
        st.largest_batch = max(st.largest_batch, k)

    def _check_margins(self, kind_ids: np.ndarray, x_rows: np.ndarray, y_rows: np.ndarray) -> None:
        bx, by = self._bounds[x_rows], self._bounds[y_rows]
        # every kind passes when both bounds are below margin / (|cx| + |cy|): the common case, two reductions
        if max(bx.max(), by.max()) < self._safe_bound:
            return
        load = self._absx[kind_ids] * bx + self._absy[kind_ids] * by
        room = self._margins[kind_ids]
        if np.any(load >= room):
            j = int(np.argmax(load - room))
            raise BootstrapMarginError(
                f"{TWO_INPUT_KINDS[int(kind_ids[j])].value}: combined noise bound {load[j]:.3g} "
                f"reaches margin {room[j]:.3g}"
            )

    def _new_rows(self, count: int) -> RowBlock:
        block = self._alloc.alloc(count)
        end = block.start + count
        if end > len(self._bounds):
            grown = np.zeros(max(end, 2 * len(self._bounds)), dtype=np.float64)
            grown[: len(self._bounds)] = self._bounds
            self._bounds = grown
        self._reserve_storage(end)
        return block

    def _handles(self, rows, owner) -> list:
        return [EncBit(self, _row=r, _owner=owner) for r in rows]

    @staticmethod
    def _rows_of(bits) -> np.ndarray:
        return np.fromiter((b.row for b in bits), dtype=np.int64, count=len(bits))

    # -- index-array evaluation API (used by the circuit layer) -------------------------
    def gate_rows(self, kind: GateKind, x_rows: np.ndarray, y_rows: np.ndarray):
        """Elementwise gate over two row arrays, one launch (split only by
        max_batch).  Returns (output rows, owners)."""
        self._check_two_input(kind)
        k = len(x_rows)
        if k == 0 or k != len(y_rows):
            raise ValueError("need equally many left and right inputs, at least one")
        self.stats.single_gates += k
        ids = np.full(k, self._kind_index[kind], dtype=np.uint8)
        return self.pool.execute_rows(self, ids, np.asarray(x_rows, np.int64), np.asarray(y_rows, np.int64))

    def compound_rows(self, kind_a: GateKind, kind_b: GateKind, x_rows: np.ndarray, y_rows: np.ndarray):
        """Two kinds on shared input pairs: one launch of 2k jobs, jobs
        interleaved (a, b, a, b, ...) like the reference
        (`encirc/engine.py:302-320`).  Returns (rows_a, rows_b, owners)."""
        self._check_two_input(kind_a)
        self._check_two_input(kind_b)
        k = len(x_rows)
        if k == 0 or k != len(y_rows):
            raise ValueError("need equally many left and right inputs, at least one")
        self.stats.compound_gates += k
        ids = np.empty(2 * k, dtype=np.uint8)
        ids[0::2] = self._kind_index[kind_a]
        ids[1::2] = self._kind_index[kind_b]
        xs2 = np.repeat(np.asarray(x_rows, np.int64), 2)
        ys2 = np.repeat(np.asarray(y_rows, np.int64), 2)
        rows, owners = self.pool.execute_rows(self, ids, xs2, ys2)
        return rows[0::2], rows[1::2], owners

    def not_rows(self, rows: np.ndarray):
        rows = np.asarray(rows, np.int64)
        self.stats.not_gates += len(rows)
        return self._negate_rows(rows)

    def trivial_row(self, value) -> int:
        return self.trivial_bit(value).row

    # -- handle-level evaluation API (the reference's) -----------------------------------
    def eval_not(self, x: EncBit) -> EncBit:
        self._check_bit(x)
        rows, owners = self.not_rows(np.array([x.row]))
        return EncBit(self, _row=rows[0], _owner=owners)

    def eval_gate(self, kind: GateKind, x: EncBit, y: EncBit | None = None) -> EncBit:
        if kind is GateKind.NOT:
            if y is not None:
                raise ValueError("NOT takes a single input")
            return self.eval_not(x)
        if y is None:
            raise ValueError(f"{kind.value} needs two inputs")
        self._check_two_input(kind)
        self._check_bit(x)
        self._check_bit(y)
        self.stats.single_gates += 1
        return self.pool.execute_batch(JobBatch((kind,), (x,), (y,)), self)[0]

    def _checked(self, xs, ys):
        xs, ys = tuple(xs), tuple(ys)
        if len(xs) == 0 or len(xs) != len(ys):
            raise ValueError("need equally many left and right inputs, at least one")
        for b in itertools.chain(xs, ys):
            self._check_bit(b)
        return xs, ys

    def eval_gate_batch(self, kind: GateKind, xs, ys) -> list:
        self._check_two_input(kind)
        xs, ys = self._checked(xs, ys)
        rows, owners = self.gate_rows(kind, self._rows_of(xs), self._rows_of(ys))
        return self._handles(rows, owners)

    def eval_compound(self, kind_a: GateKind, kind_b: GateKind, x: EncBit, y: EncBit) -> tuple:
        outs_a, outs_b = self.eval_compound_batch(kind_a, kind_b, (x,), (y,))
        return outs_a[0], outs_b[0]

    def eval_compound_batch(self, kind_a: GateKind, kind_b: GateKind, xs, ys) -> tuple:
        self._check_two_input(kind_a)
        self._check_two_input(kind_b)
        xs, ys = self._checked(xs, ys)
        ra, rb, owners = self.compound_rows(kind_a, kind_b, self._rows_of(xs), self._rows_of(ys))
        return self._handles(ra, owners), self._handles(rb, owners)

    def execute_launch(self, kinds, xs, ys, pool) -> list:
        """The scheduler-facing hook of the reference
        (`encirc/engine.py:339-340,458-514`): one launch over handle tuples."""
        ids = np.fromiter((self._kind_index[kd] for kd in kinds), dtype=np.uint8, count=len(kinds))
        rows, owners = self.launch_rows(ids, self._rows_of(xs), self._rows_of(ys))
        return self._handles(rows, owners)

    def launch_rows(self, kind_ids: np.ndarray, x_rows: np.ndarray, y_rows: np.ndarray):
        """One launch: count it, check margins, evaluate, return (rows, owners)."""
        k = len(kind_ids)
        self._count_launch(k)
        self._check_margins(kind_ids, x_rows, y_rows)
        block = self._new_rows(k)
        out_rows = block.rows()
        self._submit(kind_ids, x_rows, y_rows, out_rows)
        self._bounds[block.start : block.start + k] = self.fresh_bound
        return out_rows, (block,)

    # -- levelised execution ---------------------------------------------------------------
    # The reference issues one launch per circuit step (`encirc/scheduler.py:156-171`): three per bit of
    # a ripple-carry adder (`encirc/integers.py:95-113`), one adder after the other through the levels of
    # a multiplier tree (`encirc/integers.py:177-238`).  A real bootstrap is deterministic, so WHEN a
    # launch runs is invisible: a lazy engine counts and checks every launch at the call (statistics,
    # margins and errors are the reference's) but only records it, with its LEVEL = 1 + the highest level
    # among the still-unevaluated launches that produce its inputs.  When something reads a row (a
    # decryption, a NOT, a serialisation) or the queue holds MAX_DEFERRED_GATES, the queue runs level by
    # level, all launches of a level -- mutually independent by construction -- as ONE kernel launch.
    # The carry-independent launches of an adder collapse into one, and the adders of consecutive tree
    # levels run as a wavefront: a 32-bit multiply is 138 dependent kernel launches instead of 961.
    lazy = False
    MAX_DEFERRED_GATES = 1 << 20      # rows stay allocated until the queue has run: 2 GiB of ciphertexts
    MAX_DEFERRED_LAUNCHES = 1 << 14

    def _submit(self, kind_ids, x_rows, y_rows, out_rows) -> None:
        if not self.lazy:
            self.physical_launches += 1
            self._evaluate(kind_ids, x_rows, y_rows, out_rows)
            return
        x_rows = np.array(x_rows, np.int64)
        y_rows = np.array(y_rows, np.int64)
        out_rows = np.array(out_rows, np.int64)
        k = len(kind_ids)
        if self._deferred and (self._deferred_gates + k > self.MAX_DEFERRED_GATES
                               or self._deferred_launches >= self.MAX_DEFERRED_LAUNCHES):
            self._run_deferred()
        if len(self._row_level) < len(self._bounds):
            grown = np.zeros(len(self._bounds), dtype=np.int32)
            grown[: len(self._row_level)] = self._row_level
            self._row_level = grown
        # levels are absolute depths of the current queue epoch: levels up to _depth_done have already been handed
        # to the device (early start, below), so a launch whose inputs are all evaluated joins the next one to run
        level = self._depth_done + 1
        if self._deferred:
            lv = self._row_level
            level = max(level, 1 + int(max(lv[x_rows].max(), lv[y_rows].max())))
        self._alloc.hold = True  # rows freed from now on may still be read or written by the queue
        self._deferred.setdefault(level, []).append((np.array(kind_ids, np.uint8), x_rows, y_rows, out_rows))
        self._deferred_gates += k
        self._deferred_launches += 1
        self._row_level[out_rows] = level
        self._early_start()

    def _early_start(self) -> None:
        """Hook: an engine whose device would otherwise idle while a circuit is still being recorded may hand the
        lowest queued level over now (`_run_next_level`).  Default: nothing runs before something reads a row."""

    def _run_next_level(self) -> None:
        """Execute the lowest queued level as one kernel launch; everything above it stays queued."""
        level = min(self._deferred)
        batch = self._deferred.pop(level)
        gates = sum(len(q[0]) for q in batch)
        try:
            if len(batch) == 1:
                kinds, xs, ys, outs = batch[0]
            else:
                kinds, xs, ys, outs = (np.concatenate([q[j] for q in batch]) for j in range(4))
            self.physical_launches += 1
            self._evaluate(kinds, xs, ys, outs)
        finally:
            for q in batch:
                self._row_level[q[3]] = 0
            self._deferred_gates -= gates
            self._deferred_launches -= len(batch)
            self._depth_done = level
            if not self._deferred:  # the epoch is over: depths start again, quarantined rows go back to the allocator
                self._depth_done = 0
                self._alloc.end_hold()

    def _run_deferred(self) -> None:
        """Execute the queue, one kernel launch per level.  Called before anything reads or rewrites rows."""
        try:
            while self._deferred:
                self._run_next_level()
        except BaseException:
            # after an error nothing may stay marked as pending
            for batch in self._deferred.values():
                for q in batch:
                    self._row_level[q[3]] = 0
            self._deferred = {}
            self._deferred_gates = self._deferred_launches = 0
            self._depth_done = 0
            self._alloc.end_hold()
            raise

    def bootstrap(self, bit: EncBit) -> EncBit:
        """Standalone refresh; precondition noise_bound < mu, one launch."""
        self._check_bit(bit)
        mu = self.params.mu_float
        if bit.noise_bound >= mu:
            raise BootstrapMarginError(f"noise_bound {bit.noise_bound:.3g} >= margin {mu:.3g}")
        self._count_launch(1)
        block = self._new_rows(1)
        self._refresh(np.array([bit.row], np.int64), block.rows())
        self._bounds[block.start] = self.fresh_bound
        return EncBit(self, _row=block.start, _owner=(block,))

    def trivial_bit(self, value) -> EncBit:
        v = _bit_value(value)
        bit = self._trivial.get(v)
        if bit is None:
            block = self._new_rows(1)
            self._store_trivial(block.start, v)
            self._bounds[block.start] = 0.0
            bit = self._trivial[v] = EncBit(self, _row=block.start, _owner=(block,))
        return bit

    def encrypt(self, value) -> EncBit:
        rows, owners = self.encrypt_rows([_bit_value(value)])
        return EncBit(self, _row=rows[0], _owner=owners)

    def decrypt(self, bit: EncBit) -> int:
        self._check_bit(bit)
        return int(self.decrypt_rows(np.array([bit.row], np.int64))[0])

    def _check_decryptable(self, rows: np.ndarray) -> None:
        limit = self.params.mu_float / 2
        worst = float(self._bounds[rows].max())
        if worst >= limit:
            raise DecryptionUnreliableError(f"noise_bound {worst:.3g} >= mu/2 = {limit:.3g}")

    # -- engine-specific hooks ------------------------------------------------------------
    def _reserve_storage(self, rows: int) -> None:
        raise NotImplementedError

    def _evaluate(self, kind_ids, x_rows, y_rows, out_rows) -> None:
        raise NotImplementedError

    def _refresh(self, in_rows, out_rows) -> None:
        raise NotImplementedError

    def _negate_rows(self, rows):
        raise NotImplementedError

    def _store_trivial(self, row: int, value: int) -> None:
        raise NotImplementedError

    def encrypt_rows(self, values):
        raise NotImplementedError

    def decrypt_rows(self, rows) -> np.ndarray:
        raise NotImplementedError

    def _adopt(self, sample, clear, bound):
        raise NotImplementedError

    def _row_sample(self, row: int):
        return None

    def _row_clear(self, row: int):
        return None


class ReferenceEngine(GateEngine):
    """Cleartext engine with full phantom accounting: same stats, noise-bound
    bookkeeping and margin errors as an LWE engine, no ciphertexts
    (reference `encirc/engine.py:343-402`)."""

    name = "reference"

    def __init__(self, params: LweParams | None = None, pool: WorkerPool | None = None, seed: int = 0):
        self._clear = np.zeros(1024, dtype=np.uint8)
        super().__init__(params if params is not None else LweParams(), pool)
        self.seed = int(seed)  # draws no randomness; kept so callers derive input streams uniformly

    def _reserve_storage(self, rows: int) -> None:
        if rows > len(self._clear):
            grown = np.zeros(max(rows, 2 * len(self._clear)), dtype=np.uint8)
            grown[: len(self._clear)] = self._clear
            self._clear = grown

    def _evaluate(self, kind_ids, x_rows, y_rows, out_rows) -> None:
        self._clear[out_rows] = self._truth[kind_ids, (self._clear[x_rows] << 1) | self._clear[y_rows]]

    def _refresh(self, in_rows, out_rows) -> None:
        self._clear[out_rows] = self._clear[in_rows]

    def _negate_rows(self, rows):
        block = self._new_rows(len(rows))
        out = block.rows()
        self._clear[out] = 1 - self._clear[rows]
        self._bounds[out] = self._bounds[rows]
        return out, (block,)

    def _store_trivial(self, row: int, value: int) -> None:
        self._clear[row] = value

    def encrypt_rows(self, values):
        vals = np.asarray([_bit_value(v) for v in values], dtype=np.uint8)
        block = self._new_rows(len(vals))
        out = block.rows()
        self._clear[out] = vals
        self._bounds[out] = self.fresh_bound
        return out, (block,)

    def decrypt_rows(self, rows) -> np.ndarray:
        rows = np.asarray(rows, np.int64)
        self._check_decryptable(rows)
        return self._clear[rows].astype(np.int64)

    def _adopt(self, sample, clear, bound):
        if sample is not None or clear is None:
            raise ValueError("the cleartext engine adopts clear bits only")
        block = self._new_rows(1)
        self._clear[block.start] = _bit_value(clear)
        self._bounds[block.start] = 0.0 if bound is None else float(bound)
        return block.start, (block,)

    def _row_clear(self, row: int):
        return int(self._clear[row])


class B200Engine(GateEngine):
    """Real TFHE gate bootstrapping on one B200 through libtfhe_b200.so.

    Takes the place of the reference's `OracleBootstrapEngine`
    (`encirc/engine.py:405-514`): same constructor shape `(key, seed, pool)`,
    same encryption stream `default_rng((seed, 0))` so fresh ciphertexts are
    word-for-word those of the reference, same stats, margins and errors.  The
    bootstrap itself is the real thing: linear form -> blind rotation against
    the spectral bootstrapping key -> sample extract -> key switch, all on the
    device; the secret key is only used by `encrypt` / `decrypt`.

    There is no CPU fallback: constructing the engine without the CUDA
    library or without a GPU raises.
    """

    name = "b200-tfhe"
    _ENC_STREAM = 0
    lazy = os.environ.get("TFB_EAGER", "0") in ("", "0")  # TFB_EAGER=1: one kernel launch per logical launch

    def __init__(self, key: SecretKey, seed: int = 0, pool: WorkerPool | None = None, *,
                 device: int | None = None, ring=None, eval_keys=None, initial_rows: int = 1 << 16,
                 device_encrypt: bool = False, raw_key_tensors=None):
        import torch  # device memory + streams only

        from . import _cabi
        from .keys import RingParams, generate_evaluation_keys

        if key.params.w != 32:
            raise ValueError("the B200 engine works on the 32-bit torus only")
        if not torch.cuda.is_available():
            raise _cabi.TfbError("no CUDA device visible: the B200 engine has no CPU fallback")
        self._torch = torch
        self._cabi = _cabi
        self.key = key
        self.seed = int(seed)
        self.device_index = torch.cuda.current_device() if device is None else int(device)
        self.device = torch.device("cuda", self.device_index)
        self._pool_t = torch.zeros((initial_rows, _cabi.ROW_STRIDE), dtype=torch.int32, device=self.device)
        self._pending: list = []  # (first row, packed host words) awaiting upload
        self._stage = None
        self._submits = 0
        self._inflight: list = []  # completion events of levels handed to the device ahead of a flush
        super().__init__(key.params, pool)
        self._enc_rng = np.random.default_rng((self.seed, self._ENC_STREAM))
        # device_encrypt: fresh encryptions drawn on the GPU by a counter-based generator (throughput inputs:
        # 0.5 M bits of config 5 in milliseconds instead of ~11 s of host numpy).  Off by default because the
        # reference's draw order -- and with it word-for-word identity of fresh ciphertexts -- is a host stream.
        self.device_encrypt = bool(device_encrypt)
        self._enc_counter = 0
        self.ring = ring if ring is not None else RingParams()
        self._ctx = _cabi.Context(self.device_index, key.params.m, key.params.mu.word, self.ring)
        if raw_key_tensors is not None:
            # (bk, ksk) already on this device -- the receive buffers of the NCCL key broadcast
            # (sharding.broadcast_eval_keys); the device transforms them itself (kernel K3)
            bk_t, ksk_t = raw_key_tensors
            self.eval_keys = eval_keys
            self._ctx.call("tfb_load_keys", bk_t.data_ptr(), ksk_t.data_ptr(), 1, self._stream())
        else:
            self.eval_keys = eval_keys if eval_keys is not None else generate_evaluation_keys(key, self.seed, self.ring)
            self._ctx.call("tfb_load_keys", self.eval_keys.bk.ctypes.data, self.eval_keys.ksk.ctypes.data, 0,
                           self._stream())
        self._key_bits_t = torch.from_numpy(key.bits.astype(np.uint32).view(np.int32)).to(self.device)

    # -- plumbing -------------------------------------------------------------------------
    def _stream(self):
        return self._torch.cuda.current_stream(self.device).cuda_stream

    def _reserve_storage(self, rows: int) -> None:
        have = self._pool_t.shape[0]
        if rows <= have:
            return
        torch = self._torch
        grown = torch.zeros((max(rows, 2 * have), self._cabi.ROW_STRIDE), dtype=torch.int32, device=self.device)
        grown[:have] = self._pool_t
        self._pool_t = grown

    def _flush(self) -> None:
        """Bring device storage up to date: queued launches first (their inputs' uploads happen inside),
        then host words waiting for upload."""
        self._run_deferred()
        self._upload_pending()

    def _upload_pending(self) -> None:
        if not self._pending:
            return
        torch, n1 = self._torch, self.params.m + 1
        for start, words in self._pending:
            if isinstance(words, np.ndarray):
                words = torch.from_numpy(words.view(np.int32)).to(self.device)
            self._pool_t[start : start + len(words), :n1] = words
        self._pending = []

    def _dev(self, arr: np.ndarray, dtype):
        return self._torch.from_numpy(np.ascontiguousarray(arr, dtype=dtype)).to(self.device)

    # -- evaluation -------------------------------------------------------------------------
    EVAL_CHUNK = 1 << 18  # gates per tfb_gate_launch: bounds the library's extracted-sample scratch at 1.1 GB

    STAGE_GATES = 4096  # launches up to this size send their index arrays through one pinned staging copy

    def _stage_small(self, kind_ids, x_rows, y_rows, out_rows):
        """Index arrays + kinds of a narrow launch in ONE host->device copy from pinned memory (the latency path issues
        a launch per gate level: two pageable copies per level were ~5 % of a level).  Staging slots rotate; each carries
        the event of its last copy."""
        torch, k = self._torch, len(kind_ids)
        if self._stage is None:
            words = 4 * self.STAGE_GATES  # x, y, out (int32 each) + kinds (uint8, padded to a word each 4)
            self._stage = [(torch.empty(words, dtype=torch.int32).pin_memory(),
                            torch.empty(words, dtype=torch.int32, device=self.device),
                            torch.cuda.Event()) for _ in range(16)]
            self._stage_at = 0
            self._stage_used = 0
        host, dev, copied = self._stage[self._stage_at]
        self._stage_at = (self._stage_at + 1) % len(self._stage)
        if self._stage_used >= len(self._stage):
            # the pinned half of a slot may be rewritten once ITS last copy has run (sixteen launches ago: long done);
            # the device half is protected by stream order.  No stream-wide wait: the queue of levels stays full.
            copied.synchronize()
        self._stage_used += 1
        h = host.numpy()
        h[:k], h[k : 2 * k], h[2 * k : 3 * k] = x_rows, y_rows, out_rows
        h[3 * k : 3 * k + (k + 3) // 4].view(np.uint8)[:k] = kind_ids
        n = 3 * k + (k + 3) // 4
        dev[:n].copy_(host[:n], non_blocking=True)
        copied.record(torch.cuda.current_stream(self.device))
        return dev.data_ptr(), dev.data_ptr() + 12 * k

    # Early start: a circuit is recorded launch by launch (~20 us of Python each: 19 ms for a 32-bit multiply) before
    # anything reads a result, and the device would idle meanwhile.  Every eighth recorded launch the engine looks at
    # the device; while fewer than two handed-over levels are still in flight it hands over the lowest queued level.
    # Levels are absolute depths (GateEngine._submit), so launches recorded later simply join the next level to run.
    EARLY_START = os.environ.get("TFB_EARLY_START", "1") not in ("", "0")
    EARLY_START_EVERY = 8
    EARLY_START_IN_FLIGHT = 2

    def _early_start(self) -> None:
        if not self.EARLY_START:
            return
        self._submits += 1
        if self._submits % self.EARLY_START_EVERY:
            return
        inflight = self._inflight
        while inflight and inflight[0].query():
            inflight.pop(0)
        if len(inflight) < self.EARLY_START_IN_FLIGHT and self._deferred:
            self._run_next_level()
            done = self._torch.cuda.Event()
            done.record(self._torch.cuda.current_stream(self.device))
            inflight.append(done)

    def _evaluate(self, kind_ids, x_rows, y_rows, out_rows) -> None:
        self._upload_pending()  # (not _flush: the queue above this level stays queued)
        k = len(kind_ids)
        if k <= self.STAGE_GATES:
            base, kinds_ptr = self._stage_small(kind_ids, x_rows, y_rows, out_rows)
            self._ctx.call("tfb_gate_launch", self._pool_t.data_ptr(), kinds_ptr, base, base + 4 * k, base + 8 * k, k,
                           self._stream())
            return
        idx = self._dev(np.concatenate([x_rows, y_rows, out_rows]), np.int32)
        kinds = self._dev(kind_ids, np.uint8)
        base, step = idx.data_ptr(), 4 * k
        for lo in range(0, k, self.EVAL_CHUNK):  # gates of a launch are independent: chunking is unobservable
            kc = min(self.EVAL_CHUNK, k - lo)
            self._ctx.call("tfb_gate_launch", self._pool_t.data_ptr(), kinds.data_ptr() + lo, base + 4 * lo,
                           base + step + 4 * lo, base + 2 * step + 4 * lo, kc, self._stream())

    def _refresh(self, in_rows, out_rows) -> None:
        self._submit(np.full(len(in_rows), IDENTITY_KIND_ID, np.uint8), in_rows, in_rows, out_rows)

    def _negate_rows(self, rows):
        self._flush()
        block = self._new_rows(len(rows))
        out = block.rows()
        idx = self._dev(np.concatenate([rows, out]), np.int32)
        self._ctx.call("tfb_rows_negate", self._pool_t.data_ptr(), idx.data_ptr(), idx.data_ptr() + 4 * len(rows),
                       len(rows), self._stream())
        self._bounds[out] = self._bounds[rows]
        return out, (block,)

    def _store_trivial(self, row: int, value: int) -> None:
        words = np.zeros((1, self.params.m + 1), dtype=np.uint32)
        words[0, -1] = self.params.message_word(value)
        self._pending.append((row, words))

    # -- client side: encryption / decryption ------------------------------------------------
    def encrypt_rows(self, values):
        """Fresh encryptions in the reference's draw order (mask, then one
        normal deviate per bit: `encirc/torus.py:254-271`)."""
        p = self.params
        if self.device_encrypt:
            return self.encrypt_rows_device(values)
        vals = [_bit_value(v) for v in values]
        words = np.empty((len(vals), p.m + 1), dtype=np.uint32)
        noise = np.empty(len(vals), dtype=np.uint32)
        for i in range(len(vals)):
            words[i, : p.m] = uniform_words(p, self._enc_rng, p.m)
            noise[i] = gaussian_noise_words(p, self._enc_rng, 1)[0]
        msg = np.where(np.asarray(vals, dtype=bool), np.uint32(p.message_word(1)), np.uint32(p.message_word(0)))
        words[:, p.m] = words[:, : p.m] @ self.key.bits.astype(np.uint32) + msg + noise
        block = self._new_rows(len(vals))
        self._pending.append((block.start, words))
        out = block.rows()
        self._bounds[out] = self.fresh_bound
        return out, (block,)

    def encrypt_rows_device(self, values):
        """Fresh encryptions of a bit array drawn on the device (`tfb_rows_encrypt`: Philox4x32-10 keyed by
        the engine seed, sample counter continuing across calls).  Same distribution as `encrypt_rows`
        (uniform mask, rounded clipped Gaussian(alpha) noise), different draw order."""
        vals = np.asarray(values)
        if vals.size == 0 or not np.isin(vals, (0, 1)).all():
            raise ValueError("bit values must be 0 or 1, at least one")
        vals = vals.astype(np.uint8).reshape(-1)
        block = self._new_rows(len(vals))
        out = block.rows()
        self._flush()
        bits = self._dev(vals, np.uint8)
        idx = self._dev(out, np.int32)
        seed = (self.seed ^ 0x5EED0E1C0DE) & 0xFFFFFFFFFFFFFFFF
        self._ctx.call("tfb_rows_encrypt", self._pool_t.data_ptr(), idx.data_ptr(), bits.data_ptr(),
                       self._key_bits_t.data_ptr(), float(self.params.alpha), seed, self._enc_counter, len(vals),
                       self._stream())
        self._enc_counter += len(vals)
        self._bounds[out] = self.fresh_bound
        return out, (block,)

    def phases(self, rows) -> np.ndarray:
        """b - <a, s> of the given rows, computed on the device."""
        self._flush()
        rows = np.asarray(rows, np.int64)
        torch = self._torch
        idx = self._dev(rows, np.int32)
        out = torch.empty(len(rows), dtype=torch.int32, device=self.device)
        self._ctx.call("tfb_rows_phase", self._pool_t.data_ptr(), idx.data_ptr(), self._key_bits_t.data_ptr(),
                       out.data_ptr(), len(rows), self._stream())
        return out.cpu().numpy().view(np.uint32)

    def decrypt_rows(self, rows) -> np.ndarray:
        rows = np.asarray(rows, np.int64)
        self._check_decryptable(rows)
        ph = self.phases(rows)
        return ((ph > 0) & (ph < np.uint32(self.params.half_word))).astype(np.int64)

    def read_rows(self, rows) -> np.ndarray:
        """Packed ciphertext words [k][m+1] of the given rows (device -> host)."""
        self._flush()
        idx = self._dev(np.asarray(rows, np.int64), np.int64)
        return self._pool_t[idx, : self.params.m + 1].cpu().numpy().view(np.uint32)

    def write_rows(self, words: np.ndarray, bounds) -> tuple:
        """Adopt packed ciphertext words [k][m+1] as new rows."""
        words = np.ascontiguousarray(words, dtype=np.uint32)
        block = self._new_rows(len(words))
        self._pending.append((block.start, words))
        out = block.rows()
        self._bounds[out] = bounds
        return out, (block,)

    def adopt_words_tensor(self, t, bounds) -> tuple:
        """Adopt a device tensor [k][m+1] (int32 bit patterns) as new rows without a host round trip
        (receive buffers of the sharding collectives).  Ordered with the host uploads."""
        block = self._new_rows(t.shape[0])
        self._pending.append((block.start, t.to(device=self.device, dtype=self._torch.int32)))
        out = block.rows()
        self._bounds[out] = bounds
        return out, (block,)

    def export_words_tensor(self, rows):
        """Packed ciphertext words [k][m+1] of the given rows as a device tensor (int32 bit patterns)."""
        self._flush()
        idx = self._dev(np.asarray(rows, np.int64), np.int64)
        return self._pool_t[idx, : self.params.m + 1]

    def _adopt(self, sample, clear, bound):
        if sample is None:
            raise ValueError("an LWE engine adopts samples only")
        p = self.params
        if sample.w != p.w or len(sample.a) != p.m:
            raise ValueError("sample dimensions do not match engine parameters")
        words = np.concatenate([np.asarray(sample.a, dtype=np.uint32), [np.uint32(sample.b)]])[None, :]
        rows, owners = self.write_rows(words, sample.noise_bound)
        return int(rows[0]), owners

    def _row_sample(self, row: int):
        w = self.read_rows([row])[0]
        return LweSample(w[:-1].copy(), int(w[-1]), float(self._bounds[row]), self.params.w)

    @property
    def kernel_launches(self) -> int:
        return self._ctx.kernel_launches

    def synchronize(self) -> None:
        self._flush()
        self._torch.cuda.synchronize(self.device)
