"""Worker for tests/test_sharding_gloo.py (launched by torch.distributed.run, gloo, CPU)."""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_01945_b200 import LweParams, PoolConfig, WorkerPool, decrypt_int, encrypt_int, keygen  # noqa: E402
from paper_2005_01945_b200.integers import EncryptedInt  # noqa: E402
from paper_2005_01945_b200.sharding import (  # noqa: E402
    lane_block, sharded_mat_add, sharded_mat_mul, sharded_vec_add, sharded_vec_mul,
)
from tests.host_engine import HostOracleEngine  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
params = LweParams(m=48)
key = keygen(params, seed=5)
eng = HostOracleEngine(key, seed=9, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)), lazy=True)
lanes, width = 5, 3  # ragged on purpose: 5 lanes over 2 ranks
u_vals, v_vals = [1, 7, 5, 2, 6], [3, 7, 4, 0, 1]
a_vals, b_vals = [[1, 2, 3], [3, 0, 1], [2, 2, 1]], [[1, 0, 2], [3, 1, 1], [0, 2, 3]]  # 3x3: 9 cells over 2 ranks


def pack(values):
    if rank != 0:
        return None
    return np.stack([eng.read_rows(encrypt_int(eng, v, width)._rows) for v in values])


u_words, v_words = pack(u_vals), pack(v_vals)
a_words, b_words = pack([v for row in a_vals for v in row]), pack([v for row in b_vals for v in row])
report = {"rank": rank, "block": list(lane_block(lanes, world, rank))}
for name, call in (
    ("add", lambda: sharded_vec_add(eng, u_words, v_words, lanes, width, with_stats=True)),
    ("mul", lambda: sharded_vec_mul(eng, u_words, v_words, lanes, width, with_stats=True)),
    ("mat_add", lambda: sharded_mat_add(eng, a_words, b_words, 3, 3, width, with_stats=True)),
    ("mat_mul", lambda: sharded_mat_mul(eng, a_words, b_words, 3, 3, 3, width, with_stats=True)),
):
    eng.reset_stats()
    words, logical = call()
    report[name + "_stats"] = eng.stats.as_record()      # this rank's own counters
    report[name + "_logical"] = logical.as_record()      # merged: the unsharded circuit's
    if rank == 0:
        out = []
        for lane in words:
            rows, owners = eng.write_rows(lane, eng.fresh_bound)
            out.append(decrypt_int(eng, EncryptedInt._wrap(eng, rows, owners)))
        report[name] = out
    else:
        assert words is None
print("REPORT " + json.dumps(report), flush=True)
dist.barrier()
dist.destroy_process_group()
