"""Profiling target (not a pytest module): `--reps` launches of `--k` NAND gates
through tfb_gate_launch, for `ncu` to attach to.  Example (under gpurun):
  ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap -s 1 -c 1 \
      -o gpurun_out/k1 python tests/gpu_profile_target.py --k 2368 --reps 2
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2005_01945_b200 import LweParams, _cabi, generate_evaluation_keys, keygen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=2368)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
dev = torch.device("cuda:0")
key = keygen(LweParams(), seed=bench.KEY_SEED)
ek = generate_evaluation_keys(key, seed=bench.ENGINE_SEED)
n, k = key.params.m, args.k
ctx = _cabi.Context(0, n, key.params.mu.word, ek.ring)
ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
bits, words = bench.synth_inputs(key.bits, k, 1)
pool = torch.zeros((3 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
pool[:k, : n + 1] = torch.from_numpy(words[0].view(np.int32)).to(dev)
pool[k : 2 * k, : n + 1] = torch.from_numpy(words[1].view(np.int32)).to(dev)
kinds = torch.full((k,), bench.NAND, dtype=torch.uint8, device=dev)
idx = torch.arange(3 * k, dtype=torch.int32, device=dev)
for _ in range(args.reps):
    ctx.call("tfb_gate_launch", pool.data_ptr(), kinds.data_ptr(), idx[:k].data_ptr(), idx[k : 2 * k].data_ptr(),
             idx[2 * k :].data_ptr(), k, None)
torch.cuda.synchronize()
print("profiled", args.reps, "launches of", k, "gates;", ctx.kernel_launches, "kernels")
