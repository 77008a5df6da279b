"""Launch scheduler: splitting, slot scatter, reentry guard, tree levels
(behaviours of reference encirc/scheduler.py:143-212)."""
import math
import os

import numpy as np
import pytest

from paper_2005_01945_b200 import DEFAULT_MAX_BATCH, GateKind, JobBatch, PoolConfig, WorkerPool


class LaunchRecorder:
    """Duck-typed backend: only execute_launch, like the reference's scheduler test."""

    def __init__(self):
        self.sizes = []

    def execute_launch(self, kinds, xs, ys, pool):
        self.sizes.append(len(kinds))
        return [(k, x, y) for k, x, y in zip(kinds, xs, ys)]


def test_defaults_and_env(monkeypatch):
    assert PoolConfig().max_batch == DEFAULT_MAX_BATCH == 4096
    assert PoolConfig().workers == (os.cpu_count() or 1)
    monkeypatch.setenv("WORKERS", "3")
    monkeypatch.setenv("MAX_BATCH", "77")
    assert (PoolConfig.from_env().workers, PoolConfig.from_env().max_batch) == (3, 77)
    assert PoolConfig.from_env(workers=5).workers == 5  # explicit beats env
    monkeypatch.setenv("WORKERS", "many")
    with pytest.raises(ValueError):
        PoolConfig.from_env()
    with pytest.raises(ValueError):
        PoolConfig(workers=0)
    with pytest.raises(ValueError):
        PoolConfig(max_batch=0)


def test_launch_splitting_and_order():
    pool = WorkerPool(PoolConfig(workers=1, max_batch=32))
    rec = LaunchRecorder()
    batch = JobBatch([GateKind.AND] * 100, range(100), range(100, 200))
    outs = pool.execute_batch(batch, rec)
    assert rec.sizes == [32, 32, 32, 4]
    assert [o[1] for o in outs] == list(range(100))


def test_slot_scatter_and_validation():
    pool = WorkerPool(PoolConfig(workers=1, max_batch=2))
    rec = LaunchRecorder()
    outs = pool.execute_batch(JobBatch([GateKind.OR] * 3, "abc", "xyz", slots=[2, 0, 1]), rec)
    assert [o[1] for o in outs] == ["b", "c", "a"]
    with pytest.raises(ValueError):
        JobBatch([], [], [])
    with pytest.raises(ValueError):
        JobBatch([GateKind.OR] * 2, "ab", "x")
    with pytest.raises(ValueError):
        JobBatch([GateKind.OR] * 2, "ab", "xy", slots=[0, 0])
    with pytest.raises(ValueError):
        JobBatch([GateKind.OR] * 2, "ab", "xy", slots=[0, 2])


def test_reentry_is_rejected():
    pool = WorkerPool(PoolConfig(workers=2))
    rec = LaunchRecorder()

    def block(i):
        return pool.execute_batch(JobBatch([GateKind.OR], "a", "b"), rec)

    with pytest.raises(RuntimeError):
        pool.run_blocks(block, 4)
    pool.shutdown()


def test_run_blocks_ordered_for_any_worker_count():
    for workers in (1, 4):
        pool = WorkerPool(PoolConfig(workers=workers))
        assert pool.run_blocks(lambda i: i * i, 9) == [i * i for i in range(9)]
        pool.shutdown()


def test_tree_levels_and_fold_equivalence():
    pool = WorkerPool(PoolConfig(workers=1))
    for k in range(1, 65):
        total = pool.parallel_reduce(list(range(k)), combine=lambda a, b: a + b)
        assert total == k * (k - 1) // 2
        assert pool.level_counter() == (math.ceil(math.log2(k)) if k > 1 else 0)
    merged = pool.parallel_reduce([1, 2, 3, 4, 5], level_combine=lambda ls, rs: [a * b for a, b in zip(ls, rs)])
    assert merged == 120
    with pytest.raises(ValueError):
        pool.parallel_reduce([])
    with pytest.raises(ValueError):
        pool.parallel_reduce([1, 2])
    with pytest.raises(ValueError):
        pool.parallel_reduce([1, 2, 3, 4], level_combine=lambda ls, rs: [0])


def test_execute_rows_splits_like_execute_batch(ref):
    pool = WorkerPool(PoolConfig(workers=1, max_batch=32))
    from paper_2005_01945_b200 import ReferenceEngine

    eng = ReferenceEngine(pool=pool)
    rows, owners = eng.encrypt_rows([i % 2 for i in range(100)])
    out, own2 = eng.gate_rows(GateKind.XOR, rows, rows[::-1].copy())
    assert eng.stats.batch_launches == 4 and eng.stats.largest_batch == 32 and eng.stats.bootstraps == 100
    assert eng.decrypt_rows(out).tolist() == [(i % 2) ^ ((99 - i) % 2) for i in range(100)]
