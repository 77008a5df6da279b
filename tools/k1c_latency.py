"""Latency of one bootstrap (blind rotation only) on the latency kernel K1e (one gate per two-SM cluster) and, for
comparison, one wave of the throughput kernel K1d, k gates per launch, checked word for word against the CPU oracle.
    python tools/k1c_latency.py [lib.so]"""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1: os.environ["TFB_LIB"] = os.path.abspath(sys.argv[1])
import torch
from paper_2005_01945_b200 import _cabi
from paper_2005_01945_b200.keys import generate_evaluation_keys
from paper_2005_01945_b200.torus import LweParams, encrypt_bit, keygen
from oracle import tfhe_oracle as orc
p = LweParams(); key = keygen(p, seed=11); ek = generate_evaluation_keys(key, seed=11); n = p.m
rng = np.random.default_rng((11, 0))
def pack(s): return np.concatenate([s.a, [s.b]]).astype(np.uint32)
K = 8
xs = np.stack([pack(encrypt_bit(key, (g >> 1) & 1, rng)) for g in range(K)])
ys = np.stack([pack(encrypt_bit(key, g & 1, rng)) for g in range(K)])
kinds = np.array([g % 8 for g in range(K)], dtype=np.uint8)
_, want = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, ek.bk, ek.ksk, want_ext=True)
dev = torch.device("cuda:0")
for which, name in (("5", "K1e k_gate_bootstrap_pair"), ("4", "K1d k_gate_bootstrap_warp")):
    os.environ["TFB_FORCE_KERNEL"] = which
    ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
    ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
    for k in (1, 2, 64, 74, 148):
        idx = torch.arange(k, device=dev) % K
        pool = torch.zeros((2 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
        pool[:k, : n + 1] = torch.from_numpy(xs.view(np.int32)).to(dev)[idx]
        pool[k:, : n + 1] = torch.from_numpy(ys.view(np.int32)).to(dev)[idx]
        kd = torch.from_numpy(kinds).to(dev)[idx].contiguous()
        xr = torch.arange(0, k, dtype=torch.int32, device=dev); yr = torch.arange(k, 2 * k, dtype=torch.int32, device=dev)
        ext = torch.zeros((k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)
        run = lambda: ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), ext.data_ptr(), k, None)
        run(); torch.cuda.synchronize()
        bad = int((ext.cpu().numpy().view(np.uint32)[:, :1025] != want[np.arange(k) % K]).sum())
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): run()
        e1.record(); torch.cuda.synchronize()
        print(f"{name}  k={k:4d}  {e0.elapsed_time(e1) / 20:.4f} ms per launch  mismatch_words={bad}", flush=True)
    ctx.close()
