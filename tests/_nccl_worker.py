"""Worker for tests/test_gpu_sharding.py: the sharding code over the NCCL backend (one rank per visible GPU; the
GPU box has one, so world size 1 -- every collective still executes, on device tensors)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_01945_b200 import (  # noqa: E402
    B200Engine, LweParams, PoolConfig, ReferenceEngine, WorkerPool, encrypt_matrix, encrypt_vector, keygen, mat_add,
    mat_mul_flat, vec_add, vec_mul,
)
from paper_2005_01945_b200 import sharding  # noqa: E402

rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
key = keygen(LweParams(), seed=11)
eng = B200Engine(key, seed=11, device=local, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)))
width, lanes, q = 6, 7, 3
rng = np.random.default_rng(5)
u, v = (rng.integers(0, 1 << width, size=lanes).tolist() for _ in range(2))
a, b = (rng.integers(0, 1 << width, size=(q, q)).tolist() for _ in range(2))


def pack_dev(ints):
    """Packed operand words as a DEVICE tensor on the root (what a sharded caller hands over)."""
    if rank != 0:
        return None
    rows = np.concatenate([x._rows for x in ints])
    return eng.export_words_tensor(rows).reshape(len(ints), width, -1).clone()


def logical(circuit):
    ref = ReferenceEngine(pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)))
    circuit(ref)
    return ref.stats.as_record()


U, V = encrypt_vector(eng, u, width), encrypt_vector(eng, v, width)
A, B = encrypt_matrix(eng, a, width), encrypt_matrix(eng, b, width)
uw, vw, aw, bw = pack_dev(U.items), pack_dev(V.items), pack_dev(A.data), pack_dev(B.data)
report = {"rank": rank, "backend": dist.get_backend(), "world": world}
cases = (
    ("vec_add", lambda: sharding.sharded_vec_add(eng, uw, vw, lanes, width, as_numpy=False, with_stats=True),
     lambda e: vec_add(encrypt_vector(e, u, width), encrypt_vector(e, v, width)), lambda: vec_add(U, V).items, width),
    ("vec_mul", lambda: sharding.sharded_vec_mul(eng, uw, vw, lanes, width, as_numpy=False, with_stats=True),
     lambda e: vec_mul(encrypt_vector(e, u, width), encrypt_vector(e, v, width)), lambda: vec_mul(U, V).items, 2 * width),
    ("mat_add", lambda: sharding.sharded_mat_add(eng, aw, bw, q, q, width, as_numpy=False, with_stats=True),
     lambda e: mat_add(encrypt_matrix(e, a, width), encrypt_matrix(e, b, width)), lambda: mat_add(A, B).data, width),
    ("mat_mul", lambda: sharding.sharded_mat_mul(eng, aw, bw, q, q, q, width, as_numpy=False, with_stats=True),
     lambda e: mat_mul_flat(encrypt_matrix(e, a, width), encrypt_matrix(e, b, width)), lambda: mat_mul_flat(A, B).data, width),
)
for name, sharded, on_ref, direct, out_width in cases:
    eng.reset_stats()
    words, stats = sharded()
    rec = {"logical_equal": stats.as_record() == logical(on_ref)}
    if rank == 0:
        rec["on_device"] = bool(words.is_cuda)
        got = words.cpu().numpy().view(np.uint32)
        want = np.stack([eng.read_rows(x._rows) for x in direct()])  # the unsharded circuit on the same engine
        rec["words_equal_unsharded"] = bool(np.array_equal(got, want))
        ph = got[..., -1] - got[..., :-1] @ key.bits.astype(np.uint32)
        bits = ((ph > 0) & (ph < 2**31)).astype(np.int64)
        rec["values"] = [int(sum(int(bit) << i for i, bit in enumerate(lane))) for lane in bits]
    report[name] = rec
report["truth"] = {
    "vec_add": [(x + y) % (1 << width) for x, y in zip(u, v)], "vec_mul": [x * y for x, y in zip(u, v)],
    "mat_add": [(a[i][j] + b[i][j]) % (1 << width) for i in range(q) for j in range(q)],
    "mat_mul": [sum(a[i][t] * b[t][j] for t in range(q)) % (1 << width) for i in range(q) for j in range(q)],
}
print("REPORT " + json.dumps(report), flush=True)
dist.barrier()
dist.destroy_process_group()
