"""The sharding module over NCCL on the GPU box (world size = visible GPUs; 1 there): scatter / broadcast / gather run
on device tensors, results equal the unsharded circuit word for word, logical GateStats equal the unsharded counts."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_sharded_ops_over_nccl():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "_nccl_worker.py")]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    rep = next(json.loads(line.split("REPORT ", 1)[1]) for line in proc.stdout.splitlines() if "REPORT " in line)
    assert rep["backend"] == "nccl"
    for name in ("vec_add", "vec_mul", "mat_add", "mat_mul"):
        rec = rep[name]
        assert rec["on_device"] and rec["logical_equal"] and rec["words_equal_unsharded"], (name, rec)
        assert rec["values"] == rep["truth"][name], name
