"""A/B timing of the K1 variants (blind rotation only) with a parity check against the CPU oracle.
    python tools/k1_ab.py [--k 16384] [--kernels 2,4] [--lib path/to/libtfhe_b200.so]
Each variant runs in this process with TFB_FORCE_KERNEL set before its context is created."""
import argparse, json, os, sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--k", default="16384", help="comma-separated launch sizes")
ap.add_argument("--kernels", default="2,4")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--lib", default=None)
args = ap.parse_args()
if args.lib:
    os.environ["TFB_LIB"] = os.path.abspath(args.lib)

import torch
from paper_2005_01945_b200 import _cabi
from paper_2005_01945_b200.keys import generate_evaluation_keys
from paper_2005_01945_b200.torus import LweParams, encrypt_bit, keygen
from oracle import tfhe_oracle as orc

dev = torch.device("cuda:0")
p = LweParams()
key = keygen(p, seed=11)
ek = generate_evaluation_keys(key, seed=11)
n = p.m
rng = np.random.default_rng((11, 0))


def pack(s):
    return np.concatenate([s.a, [s.b]]).astype(np.uint32)


K = 16
xs = np.stack([pack(encrypt_bit(key, (g >> 1) & 1, rng)) for g in range(K)])
ys = np.stack([pack(encrypt_bit(key, g & 1, rng)) for g in range(K)])
kinds = np.array([(g // 4) % 8 for g in range(K)], dtype=np.uint8)
_, want_ext = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, ek.bk, ek.ksk, want_ext=True)
res = {}
for which, k in [(w, int(kk)) for kk in args.k.split(",") for w in args.kernels.split(",")]:
    os.environ["TFB_FORCE_KERNEL"] = which
    ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
    ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
    pool = torch.zeros((2 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
    idx = torch.arange(k, device=dev) % K
    pool[:k, : n + 1] = torch.from_numpy(xs.view(np.int32)).to(dev)[idx]
    pool[k:, : n + 1] = torch.from_numpy(ys.view(np.int32)).to(dev)[idx]
    kd = torch.from_numpy(kinds).to(dev)[idx].contiguous()
    xr = torch.arange(0, k, dtype=torch.int32, device=dev)
    yr = torch.arange(k, 2 * k, dtype=torch.int32, device=dev)
    ext = torch.zeros((k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)

    def run():
        ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), ext.data_ptr(), k, None)

    run()
    torch.cuda.synchronize()
    got = ext.cpu().numpy().view(np.uint32)[:, :1025]
    bad = int((got != want_ext[np.arange(k) % K]).sum())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    res[f"{which}@{k}"] = {"ms": ms, "gates_per_s": k / ms * 1e3, "mismatch_words": bad}
    print(which, k, res[f"{which}@{k}"], flush=True)
    ctx.close()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "k1_ab.json"), "w") as f:
    json.dump(res, f)
