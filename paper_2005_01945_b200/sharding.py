"""Sharding of element-wise vector / matrix circuits and matrix products across GPUs.

One process per GPU (`torch.distributed`: NCCL over NVLink on the GPU box, gloo in the CPU tests).
Every lane of `vec_add` / `vec_mul` / `mat_add` and every output cell of a matrix product is independent
of every other at every circuit step (reference `encirc/integers.py:95-113,206-238`,
`encirc/linalg.py:156-201`), so the path shards by contiguous blocks of lanes / output cells with NO
data-path collective.  Collectives do exactly two things:

* distribute the operand ciphertexts from the root -- `dist.scatter` of each rank's lane block for the
  element-wise ops, `dist.broadcast` of both operand matrices for the matrix product (every rank needs
  whole rows of A and columns of B; 2 x 256 x 16 x 2 KB = 16 MB at 16 x 16 x 16-bit);
* `dist.gather` the result ciphertexts to the root.

The tensors stay on the device end to end: the engine adopts a received buffer straight into its row pool
(`adopt_words_tensor`) and exports result rows as a device tensor (`export_words_tensor`); nothing goes
through `.cpu()` on the NCCL path.  Evaluation keys are broadcast once by the caller (bench.py).

Statistics: a sharded operation reports the LOGICAL counters of the unsharded circuit (`merge_stats`):
launch counts do not depend on the lane count, so they are the per-rank launch count; bootstraps and gate
counts add up over the ranks; the widest logical launch is the union of the ranks' widest launches.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .engine import GateStats
from .integers import EncryptedInt, _add_lanes, _level_add, _mul_lanes, truncate


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


def _single(group=None) -> bool:
    """No process group: plain local execution.  An initialised group of ONE rank still goes through the
    collectives (that is how the NCCL path is exercised on a one-GPU box)."""
    dist = _dist()
    return not (dist.is_available() and dist.is_initialized())


def _comm_device(engine):
    """Collectives run where the ciphertexts live: the engine's GPU under NCCL, host memory under gloo."""
    import torch

    dist = _dist()
    if dist.is_initialized():
        if dist.get_backend() == "nccl":
            return getattr(engine, "device", torch.device("cuda"))
        return torch.device("cpu")
    # a single process without a process group: nothing is communicated, the words stay where the engine keeps them
    return getattr(engine, "device", torch.device("cpu"))


def _as_tensor(words, device):
    """Packed ciphertext words (numpy uint32 / int32, or a tensor) -> int32 tensor on `device`."""
    import torch

    if isinstance(words, torch.Tensor):
        return words.to(device=device, dtype=torch.int32)
    return torch.from_numpy(np.ascontiguousarray(words, dtype=np.uint32).view(np.int32)).to(device)


# -- engine <-> tensor --------------------------------------------------------------------------------
# B200Engine implements adopt_words_tensor / export_words_tensor on the device; any other row engine
# (the host stand-in of the CPU tests) goes through its numpy read_rows / write_rows.


def _adopt(engine, t) -> list:
    """Tensor [L][width][m+1] -> L EncryptedInt of this rank's engine."""
    L, width, m1 = t.shape
    if L == 0:
        return []
    flat = t.reshape(L * width, m1)
    if hasattr(engine, "adopt_words_tensor"):
        rows, owners = engine.adopt_words_tensor(flat, engine.fresh_bound)
    else:
        rows, owners = engine.write_rows(flat.cpu().numpy().view(np.uint32), engine.fresh_bound)
    return [EncryptedInt._wrap(engine, rows[i * width : (i + 1) * width], owners) for i in range(L)]


def _export(engine, items: Sequence[EncryptedInt], width: int, device):
    import torch

    m1 = engine.params.m + 1
    if not items:
        return torch.empty((0, width, m1), dtype=torch.int32, device=device)
    rows = np.concatenate([v._rows for v in items])
    if hasattr(engine, "export_words_tensor"):
        flat = engine.export_words_tensor(rows).to(device)
    else:
        flat = torch.from_numpy(engine.read_rows(rows).view(np.int32)).to(device)
    return flat.reshape(len(items), width, m1)


# -- collectives ----------------------------------------------------------------------------------------


def scatter_lanes(engine, words, lanes: int, width: int, root: int = 0, group=None):
    """Root holds packed ciphertext words [lanes][width][m+1] (numpy or tensor); every rank receives its
    own lane block as a tensor on the communication device.  `dist.scatter` with equal-sized (padded) parts:
    a rank receives lanes/world of the operand, not the whole of it."""
    import torch

    world, rank = _world(group)
    dev = _comm_device(engine)
    m1 = engine.params.m + 1
    lo, hi = lane_block(lanes, world, rank)
    if _single(group):
        return _as_tensor(words, dev)[lo:hi]
    blocks = [lane_block(lanes, world, r) for r in range(world)]
    biggest = max(b - a for a, b in blocks)
    mine = torch.empty((biggest, width, m1), dtype=torch.int32, device=dev)
    parts = None
    if rank == root:
        full = _as_tensor(words, dev)
        parts = []
        for a, b in blocks:
            part = torch.zeros((biggest, width, m1), dtype=torch.int32, device=dev)
            part[: b - a] = full[a:b]
            parts.append(part)
    _dist().scatter(mine, scatter_list=parts, src=root, group=group)
    return mine[: hi - lo]


def broadcast_words(engine, words, shape: tuple, root: int = 0, group=None):
    """Root's packed words (any leading shape) replicated on every rank."""
    import torch

    world, rank = _world(group)
    dev = _comm_device(engine)
    if _single(group):
        return _as_tensor(words, dev).reshape(shape)
    buf = _as_tensor(words, dev).reshape(shape).contiguous() if rank == root else torch.empty(
        shape, dtype=torch.int32, device=dev)
    _dist().broadcast(buf, root, group=group)
    return buf


def gather_lanes(engine, local, lanes: int, root: int = 0, group=None):
    """Inverse of scatter_lanes: the root returns the tensor [lanes][width][m+1], every other rank None.
    `dist.gather` to the root only (nobody else needs the result)."""
    import torch

    world, rank = _world(group)
    if _single(group):
        return local
    blocks = [lane_block(lanes, world, r) for r in range(world)]
    biggest = max(b - a for a, b in blocks)
    mine = torch.zeros((biggest, *local.shape[1:]), dtype=torch.int32, device=local.device)
    mine[: local.shape[0]] = local
    parts = [torch.empty_like(mine) for _ in range(world)] if rank == root else None
    _dist().gather(mine, gather_list=parts, dst=root, group=group)
    if rank != root:
        return None
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, blocks)])


def broadcast_eval_keys(key, seed: int, device, ring=None, root: int = 0, group=None) -> tuple:
    """Evaluation keys generated on the root only and broadcast RAW (bk 24.6 MB, ksk 16.4 MB of int32 words) to
    every rank's GPU; each GPU turns them into its spectral / tiled layouts itself (`tfb_load_keys`, kernel K3).
    Returns the device tensors (bk, ksk) to hand to `B200Engine(raw_key_tensors=...)`."""
    import torch

    from .keys import BK_KEYS, RingParams, generate_evaluation_keys

    ring = ring if ring is not None else RingParams()
    world, rank = _world(group)
    n = key.params.m
    bk = torch.empty(((n + 1) // 2, BK_KEYS, ring.rows, 2, ring.N), dtype=torch.int32, device=device)
    ksk = torch.empty((ring.N, ring.ks_t, n + 1), dtype=torch.int32, device=device)
    if rank == root:
        ek = generate_evaluation_keys(key, seed, ring)
        bk.copy_(torch.from_numpy(ek.bk))
        ksk.copy_(torch.from_numpy(ek.ksk))
    if not _single(group):
        _dist().broadcast(bk, root, group=group)
        _dist().broadcast(ksk, root, group=group)
    return bk, ksk


def merge_stats(engine, local: GateStats, group=None) -> GateStats:
    """Logical counters of the unsharded circuit from the per-rank ones (see the module docstring).
    A rank that owns no lanes issues no launches, hence MAX (not equality) for the launch count."""
    import torch

    if _single(group):
        return local.snapshot()
    dev = _comm_device(engine)
    dist = _dist()
    add = torch.tensor([local.single_gates, local.compound_gates, local.not_gates, local.bootstraps,
                        local.largest_batch], dtype=torch.int64, device=dev)
    top = torch.tensor([local.batch_launches], dtype=torch.int64, device=dev)
    dist.all_reduce(add, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(top, op=dist.ReduceOp.MAX, group=group)
    s, c, n, b, widest = (int(v) for v in add.tolist())
    return GateStats(single_gates=s, compound_gates=c, not_gates=n, bootstraps=b,
                     batch_launches=int(top.item()), largest_batch=widest)


# -- sharded operations -------------------------------------------------------------------------------


def _to_result(t, as_numpy: bool):
    if t is None or not as_numpy:
        return t
    return t.cpu().numpy().view(np.uint32)


def sharded_lane_op(engine, op: Callable, u_words, v_words, lanes: int, width: int, out_width: int,
                    root: int = 0, group=None, as_numpy: bool = True, with_stats: bool = False):
    """Run a two-operand lane circuit (`_add_lanes` / `_mul_lanes` shaped) on this rank's block of lanes.
    u_words / v_words: packed ciphertext words [lanes][width][m+1] on the root (ignored elsewhere).
    Returns the gathered result words [lanes][out_width][m+1] on the root (numpy uint32, or the device tensor
    with as_numpy=False) and None on the other ranks; with_stats=True adds the logical GateStats."""
    before = engine.stats.snapshot()
    xs = _adopt(engine, scatter_lanes(engine, u_words, lanes, width, root, group))
    ys = _adopt(engine, scatter_lanes(engine, v_words, lanes, width, root, group))
    outs = op(xs, ys) if xs else []
    out = gather_lanes(engine, _export(engine, outs, out_width, _comm_device(engine)), lanes, root, group)
    out = _to_result(out, as_numpy)
    if with_stats:
        return out, merge_stats(engine, engine.stats.delta(before), group)
    return out


def sharded_vec_add(engine, u_words, v_words, lanes: int, width: int, root: int = 0, group=None, **kw):
    """`vec_add` (encirc/linalg.py:132-136) with lanes split over the ranks."""
    return sharded_lane_op(engine, _add_lanes, u_words, v_words, lanes, width, width, root, group, **kw)


def sharded_vec_mul(engine, u_words, v_words, lanes: int, width: int, root: int = 0, group=None, **kw):
    """`vec_mul` (encirc/linalg.py:139-143) with lanes split over the ranks."""
    return sharded_lane_op(engine, _mul_lanes, u_words, v_words, lanes, width, 2 * width, root, group, **kw)


def sharded_mat_add(engine, a_words, b_words, rows: int, cols: int, width: int, root: int = 0, group=None, **kw):
    """`mat_add` (encirc/linalg.py:146-150): row-major cells are lanes."""
    return sharded_lane_op(engine, _add_lanes, a_words, b_words, rows * cols, width, width, root, group, **kw)


def sharded_mat_mul(engine, a_words, b_words, r: int, k: int, c: int, width: int, root: int = 0, group=None,
                    as_numpy: bool = True, with_stats: bool = False):
    """Matrix product C[r][c] = A[r][k] B[k][c] mod 2**width with the OUTPUT CELLS split over the ranks.

    A and B (packed words [r*k][width][m+1] and [k*c][width][m+1], row-major, on the root) are replicated
    on every rank; a rank then runs the reference's flat per-cell schedule (`mat_mul_flat`,
    encirc/linalg.py:165-201: all cell terms multiplied in one lane pass, each cell tree-sums its k products
    at width 2n, truncated to n bits) on its contiguous block of cells.  Unlike Cannon's schedule nothing
    rotates between GPUs.  The root returns [r*c][width][m+1]."""
    before = engine.stats.snapshot()
    world, rank = _world(group)
    m1 = engine.params.m + 1
    A = _adopt(engine, broadcast_words(engine, a_words, (r * k, width, m1), root, group))
    B = _adopt(engine, broadcast_words(engine, b_words, (k * c, width, m1), root, group))
    lo, hi = lane_block(r * c, world, rank)
    cells = [divmod(cell, c) for cell in range(lo, hi)]
    outs = []
    if cells:
        lefts = [A[i * k + t] for i, j in cells for t in range(k)]
        rights = [B[t * c + j] for i, j in cells for t in range(k)]
        prods = _mul_lanes(lefts, rights)
        if k > 1:
            prods = engine.pool.parallel_reduce([prods[t::k] for t in range(k)], level_combine=_level_add)
        outs = [truncate(v, width) for v in prods]
    out = gather_lanes(engine, _export(engine, outs, width, _comm_device(engine)), r * c, root, group)
    out = _to_result(out, as_numpy)
    if with_stats:
        return out, merge_stats(engine, engine.stats.delta(before), group)
    return out
