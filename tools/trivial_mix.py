"""Launches with a third of the gates on two trivial inputs (the zero padding of multiplier trees), interleaved: the
whole launch (regrouping, K1, key switch) against the same launch with regrouping switched off, checked word for word
against the CPU oracle.      python tools/trivial_mix.py [--k 56832]"""
import argparse, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser(); ap.add_argument("--k", type=int, default=56832); args = ap.parse_args()
import torch
from paper_2005_01945_b200 import _cabi
from paper_2005_01945_b200.keys import generate_evaluation_keys
from paper_2005_01945_b200.torus import LweParams, encrypt_bit, keygen
from oracle import tfhe_oracle as orc
p = LweParams(); key = keygen(p, seed=11); ek = generate_evaluation_keys(key, seed=11); n = p.m
rng = np.random.default_rng((11, 0))
pack = lambda s: np.concatenate([s.a, [s.b]]).astype(np.uint32)
B = 12
xs = np.stack([pack(encrypt_bit(key, g & 1, rng)) for g in range(B)]); ys = np.stack([pack(encrypt_bit(key, (g >> 1) & 1, rng)) for g in range(B)])
triv = np.zeros((2, n + 1), np.uint32); triv[0, -1] = p.message_word(0); triv[1, -1] = p.message_word(1)
base_x = np.concatenate([xs, triv[[0, 1, 0, 1, 1, 0]]]); base_y = np.concatenate([ys, triv[[0, 0, 1, 1, 0, 1]]])
kinds_b = (np.arange(B + 6) % 8).astype(np.uint8)
want = orc.gate_bootstrap_batch(base_x, base_y, kinds_b, p.mu.word, ek.bk, ek.ksk, fft=True)
k = args.k
real = np.arange(k) % B
mixed = np.where(np.arange(k) % 3 == 2, B + (np.arange(k) % 6), real)  # every third gate on trivial inputs
dev = torch.device("cuda:0")
for regroup in (True, False):
    os.environ["TFB_NO_REGROUP"] = "0" if regroup else "1"
    ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
    ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
    for name, sel in (("all real", real), ("a third trivial, interleaved", mixed)):
        pool = torch.zeros((3 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
        pool[:k, : n + 1] = torch.from_numpy(base_x.view(np.int32)).to(dev)[torch.from_numpy(sel).to(dev)]
        pool[k : 2 * k, : n + 1] = torch.from_numpy(base_y.view(np.int32)).to(dev)[torch.from_numpy(sel).to(dev)]
        kd = torch.from_numpy(kinds_b[sel]).to(dev)
        idx = torch.arange(3 * k, dtype=torch.int32, device=dev)
        run = lambda: ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), idx[:k].data_ptr(), idx[k : 2 * k].data_ptr(), idx[2 * k :].data_ptr(), k, None)
        run(); torch.cuda.synchronize()
        bad = int((pool[2 * k :, : n + 1].cpu().numpy().view(np.uint32) != want[sel]).sum())
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): run()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"regrouping {'on ' if regroup else 'off'}  {name:30s} {ms:8.3f} ms  {k / ms:8.1f} gates/ms  mismatch_words={bad}", flush=True)
    ctx.close()
