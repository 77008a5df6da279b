"""Lane sharding of element-wise vector / matrix circuits across GPUs.

One process per GPU (`torch.distributed`, NCCL on the GPU box, gloo in the CPU
tests).  Every lane of `vec_add` / `vec_mul` / `mat_add` and every output cell
of a matrix product is independent of every other at every circuit step
(reference `encirc/integers.py:95-113,206-238`), so the path shards by
contiguous lane blocks with NO data-path collective.  Collectives are used for
exactly two things: distributing the input ciphertext words from the root and
gathering the result words back (the evaluation keys are broadcast once by the
caller, see bench.py).  Logical gate statistics are those of the unsharded
circuit: launch counts do not depend on the lane count, bootstraps add up.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .integers import EncryptedInt, _add_lanes, _mul_lanes


def lane_block(total: int, world: int, rank: int) -> tuple:
    """[lo, hi) of the contiguous lane block owned by `rank` (sizes differ by at most one)."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad sharding arguments")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist

    return dist


def _world(group=None) -> tuple:
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _comm_device(engine):
    dist = _dist()
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return getattr(engine, "device", "cuda")
    return "cpu"


def scatter_lanes(engine, words: np.ndarray | None, lanes: int, width: int, root: int = 0, group=None) -> np.ndarray:
    """Root holds packed ciphertext words [lanes][width][m+1]; every rank
    receives its own lane block.  (Implemented as a broadcast of the whole
    operand followed by a local slice: operands are small next to the work
    they trigger -- 2 KB per bit against ~7 us of bootstrap per gate.)"""
    import torch

    world, rank = _world(group)
    m1 = engine.params.m + 1
    lo, hi = lane_block(lanes, world, rank)
    if world == 1:
        return np.ascontiguousarray(words[lo:hi])
    dev = _comm_device(engine)
    buf = torch.empty((lanes, width, m1), dtype=torch.int32, device=dev)
    if rank == root:
        buf.copy_(torch.from_numpy(np.ascontiguousarray(words, dtype=np.uint32).view(np.int32)))
    _dist().broadcast(buf, root, group=group)
    return buf[lo:hi].cpu().numpy().view(np.uint32)


def gather_lanes(engine, local_words: np.ndarray, lanes: int, root: int = 0, group=None) -> np.ndarray | None:
    """Inverse of scatter_lanes: the root returns [lanes][width][m+1], others None."""
    import torch

    world, rank = _world(group)
    if world == 1:
        return local_words
    dist = _dist()
    dev = _comm_device(engine)
    width, m1 = local_words.shape[1], local_words.shape[2]
    sizes = [lane_block(lanes, world, r) for r in range(world)]
    biggest = max(hi - lo for lo, hi in sizes)
    mine = torch.zeros((biggest, width, m1), dtype=torch.int32, device=dev)
    mine[: len(local_words)] = torch.from_numpy(np.ascontiguousarray(local_words).view(np.int32))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    if rank != root:
        return None
    out = np.concatenate([p[: hi - lo].cpu().numpy() for p, (lo, hi) in zip(parts, sizes)])
    return out.view(np.uint32)


def _adopt(engine, words: np.ndarray) -> list:
    """Packed words [L][width][m+1] -> L EncryptedInt of this rank's engine."""
    L, width, m1 = words.shape
    if L == 0:
        return []
    rows, owners = engine.write_rows(words.reshape(L * width, m1), engine.fresh_bound)
    return [EncryptedInt._wrap(engine, rows[i * width : (i + 1) * width], owners) for i in range(L)]


def _export(engine, items: Sequence[EncryptedInt], width: int) -> np.ndarray:
    m1 = engine.params.m + 1
    if not items:
        return np.empty((0, width, m1), dtype=np.uint32)
    rows = np.concatenate([v._rows for v in items])
    return engine.read_rows(rows).reshape(len(items), width, m1)


def sharded_lane_op(engine, op: Callable, u_words, v_words, lanes: int, width: int, out_width: int,
                    root: int = 0, group=None):
    """Run a two-operand lane circuit (`_add_lanes` / `_mul_lanes` shaped) on
    this rank's block of lanes.  u_words / v_words: packed ciphertext words
    [lanes][width][m+1] on the root (ignored elsewhere).  Returns the gathered
    result words [lanes][out_width][m+1] on the root, None on other ranks."""
    mine_u = scatter_lanes(engine, u_words, lanes, width, root, group)
    mine_v = scatter_lanes(engine, v_words, lanes, width, root, group)
    xs, ys = _adopt(engine, mine_u), _adopt(engine, mine_v)
    outs = op(xs, ys) if xs else []
    return gather_lanes(engine, _export(engine, outs, out_width), lanes, root, group)


def sharded_vec_add(engine, u_words, v_words, lanes: int, width: int, root: int = 0, group=None):
    """`vec_add` (encirc/linalg.py:132-136) with lanes split over the ranks."""
    return sharded_lane_op(engine, _add_lanes, u_words, v_words, lanes, width, width, root, group)


def sharded_vec_mul(engine, u_words, v_words, lanes: int, width: int, root: int = 0, group=None):
    """`vec_mul` (encirc/linalg.py:139-143) with lanes split over the ranks."""
    return sharded_lane_op(engine, _mul_lanes, u_words, v_words, lanes, width, 2 * width, root, group)
