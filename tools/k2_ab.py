"""Key switch A/B: K2 (IMAD pipe) vs K2t (tcgen05.mma kind::i8) vs K2n (narrow launches, up to 32 gates), bit-for-bit
comparison on random extracted samples and timing.   python tools/k2_ab.py [--k 65536]"""
import argparse, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--k", default="1,2,8,16,32,64,100,128,129,1000,5000,65536")
args = ap.parse_args()
import torch
from paper_2005_01945_b200 import _cabi
from paper_2005_01945_b200.keys import generate_evaluation_keys
from paper_2005_01945_b200.torus import LweParams, keygen
dev = torch.device("cuda:0")
p = LweParams(); key = keygen(p, seed=11); ek = generate_evaluation_keys(key, seed=11); n = p.m
ctxs = {}
for mode in ("1", "2", "3"):
    os.environ["TFB_FORCE_KS"] = mode
    c = _cabi.Context(0, n, p.mu.word, ek.ring)
    c.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
    ctxs[mode] = c
g = torch.Generator(device=dev); g.manual_seed(5)
for k in [int(x) for x in args.k.split(",")]:
    ext = torch.randint(-2**31, 2**31 - 1, (k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev, generator=g)
    rows = torch.arange(k, dtype=torch.int32, device=dev)
    outs = {}
    for mode, c in ctxs.items():
        pool = torch.full((k, _cabi.ROW_STRIDE), 7, dtype=torch.int32, device=dev)
        run = lambda: c.call("tfb_debug_key_switch", ext.data_ptr(), pool.data_ptr(), rows.data_ptr(), k, None)
        run(); torch.cuda.synchronize()
        outs[mode] = pool[:, : n + 1].clone()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): run()
        e1.record(); torch.cuda.synchronize()
        outs[mode + "ms"] = e0.elapsed_time(e1) / 10
    bad = int((outs["1"] != outs["2"]).sum().item()) + int((outs["1"] != outs["3"]).sum().item())
    print(f"k={k:6d}  K2 {outs['1ms']:.4f} ms  K2t {outs['2ms']:.4f} ms  K2n (K2 above 32 gates) {outs['3ms']:.4f} ms  mismatching words {bad}", flush=True)
