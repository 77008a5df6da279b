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


def test_sharded_vector_ops_world_size_2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "_gloo_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    reports = {}
    for line in proc.stdout.splitlines():
        if "REPORT " in line:
            r = json.loads(line.split("REPORT ", 1)[1])
            reports[r["rank"]] = r
    assert set(reports) == {0, 1}
    assert reports[0]["block"] == [0, 3] and reports[1]["block"] == [3, 5]
    assert reports[0]["sum"] == [(a + b) % 8 for a, b in zip([1, 7, 5, 2, 6], [3, 7, 4, 0, 1])]
    assert reports[0]["prod"] == [a * b for a, b in zip([1, 7, 5, 2, 6], [3, 7, 4, 0, 1])]
    # launch counts are those of the unsharded circuit on every rank; bootstraps add up to the whole
    for r in (0, 1):
        assert reports[r]["add_stats"]["batch_launches"] == 3 * 3
    assert reports[0]["add_stats"]["bootstraps"] + reports[1]["add_stats"]["bootstraps"] == 5 * 3 * 5
    assert reports[0]["mul_stats"]["bootstraps"] + reports[1]["mul_stats"]["bootstraps"] == 5 * (11 * 9 - 30)
