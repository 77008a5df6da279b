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
from paper_2005_01945_b200.sharding import lane_block, sharded_vec_add, sharded_vec_mul  # noqa: E402
from tests.host_engine import HostOracleEngine  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
params = LweParams(m=48)
key = keygen(params, seed=5)
eng = HostOracleEngine(key, seed=9, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)))
lanes, width = 5, 3  # ragged on purpose: 5 lanes over 2 ranks
u_vals, v_vals = [1, 7, 5, 2, 6], [3, 7, 4, 0, 1]
u_words = v_words = None
if rank == 0:
    us = [encrypt_int(eng, v, width) for v in u_vals]
    vs = [encrypt_int(eng, v, width) for v in v_vals]
    u_words = np.stack([eng.read_rows(x._rows) for x in us])
    v_words = np.stack([eng.read_rows(x._rows) for x in vs])
eng.reset_stats()
added = sharded_vec_add(eng, u_words, v_words, lanes, width)
add_stats = eng.stats.as_record()
eng.reset_stats()
multiplied = sharded_vec_mul(eng, u_words, v_words, lanes, width)
mul_stats = eng.stats.as_record()
lo, hi = lane_block(lanes, world, rank)
report = {"rank": rank, "block": [lo, hi], "add_stats": add_stats, "mul_stats": mul_stats}
if rank == 0:
    def decode(words, w):
        out = []
        for lane in words:
            rows, owners = eng.write_rows(lane, eng.fresh_bound)
            out.append(decrypt_int(eng, EncryptedInt._wrap(eng, rows, owners)))
        return out
    report["sum"] = decode(added, width)
    report["prod"] = decode(multiplied, 2 * width)
else:
    assert added is None and multiplied is None
print("REPORT " + json.dumps(report), flush=True)
dist.barrier()
dist.destroy_process_group()
