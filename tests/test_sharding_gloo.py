"""Multi-process lane sharding under gloo (world_size 2, CPU): real TFHE
bootstraps through the C oracle stand in for the GPU kernels."""
import json
import os
import socket
import subprocess
import sys

import pytest

from paper_2005_01945_b200.sharding import lane_block

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_lane_blocks_partition_exactly():
    for total in (0, 1, 5, 16, 4096):
        for world in (1, 2, 3, 8):
            blocks = [lane_block(total, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [hi - lo for lo, hi in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        lane_block(4, 2, 2)


def _unsharded_stats(circuit):
    """Counters of the same circuit on one cleartext engine (they are data independent)."""
    from paper_2005_01945_b200 import PoolConfig, ReferenceEngine, WorkerPool

    eng = ReferenceEngine(pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)))
    circuit(eng)
    return eng.stats.as_record()


def test_sharded_vector_and_matrix_ops_world_size_2():
    from paper_2005_01945_b200 import (
        encrypt_matrix, encrypt_vector, mat_add, mat_mul_flat, vec_add, vec_mul,
    )

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "_gloo_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    reports = {}
    for line in proc.stdout.splitlines():
        if "REPORT " in line:
            r = json.loads(line.split("REPORT ", 1)[1])
            reports[r["rank"]] = r
    assert set(reports) == {0, 1}
    assert reports[0]["block"] == [0, 3] and reports[1]["block"] == [3, 5]
    u, v = [1, 7, 5, 2, 6], [3, 7, 4, 0, 1]
    a, b = [[1, 2, 3], [3, 0, 1], [2, 2, 1]], [[1, 0, 2], [3, 1, 1], [0, 2, 3]]
    assert reports[0]["add"] == [(x + y) % 8 for x, y in zip(u, v)]
    assert reports[0]["mul"] == [x * y for x, y in zip(u, v)]
    assert reports[0]["mat_add"] == [(a[i][j] + b[i][j]) % 8 for i in range(3) for j in range(3)]
    assert reports[0]["mat_mul"] == [sum(a[i][t] * b[t][j] for t in range(3)) % 8 for i in range(3) for j in range(3)]
    # per rank: launch counts are those of the unsharded circuit, bootstraps add up to the whole
    for r in (0, 1):
        assert reports[r]["add_stats"]["batch_launches"] == 3 * 3
    assert reports[0]["add_stats"]["bootstraps"] + reports[1]["add_stats"]["bootstraps"] == 5 * 3 * 5
    assert reports[0]["mul_stats"]["bootstraps"] + reports[1]["mul_stats"]["bootstraps"] == 5 * (11 * 9 - 30)
    # merged: the LOGICAL GateStats every rank reports equal the unsharded circuit's, counter for counter
    want = {
        "add": _unsharded_stats(lambda e: vec_add(encrypt_vector(e, u, 3), encrypt_vector(e, v, 3))),
        "mul": _unsharded_stats(lambda e: vec_mul(encrypt_vector(e, u, 3), encrypt_vector(e, v, 3))),
        "mat_add": _unsharded_stats(lambda e: mat_add(encrypt_matrix(e, a, 3), encrypt_matrix(e, b, 3))),
        "mat_mul": _unsharded_stats(lambda e: mat_mul_flat(encrypt_matrix(e, a, 3), encrypt_matrix(e, b, 3))),
    }
    for name, stats in want.items():
        for r in (0, 1):
            assert reports[r][name + "_logical"] == stats, (name, r)
