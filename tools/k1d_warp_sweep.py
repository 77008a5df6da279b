"""K1d wave time against the number of gates per CTA (1 .. 12 warps), for the dispatch cost table
(TFB_K1D_WAVE_TABLE in csrc/tfhe_b200.cu): one launch of 148 * w gates, w gates on every SM, checked word for
word against the CPU oracle.  Also K1e at 74 gates (one wave).
    python tools/k1d_warp_sweep.py [lib.so]"""
import json, os, sys
import numpy as np
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
pack = lambda s: np.concatenate([s.a, [s.b]]).astype(np.uint32)
K = 16
xs = np.stack([pack(encrypt_bit(key, (g >> 1) & 1, rng)) for g in range(K)])
ys = np.stack([pack(encrypt_bit(key, g & 1, rng)) for g in range(K)])
kinds = np.array([(g // 4) % 8 for g in range(K)], dtype=np.uint8)
_, want = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, ek.bk, ek.ksk, want_ext=True)
dev = torch.device("cuda:0")
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = {}


def measure(tag, env, k, reps=5):
    for name in ("TFB_FORCE_KERNEL", "TFB_K1D_W", "TFB_K1D_NOMID"):
        os.environ.pop(name, None)
    os.environ.update(env)
    ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
    ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
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
    for _ in range(reps): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[tag] = {"k": k, "ms": ms, "gates_per_s": k / ms * 1e3, "mismatch_words": bad}
    print(tag, out[tag], flush=True)
    ctx.close()


for w in range(1, 13):
    measure(f"k1d_w{w}", {"TFB_FORCE_KERNEL": "4", "TFB_K1D_W": str(w)}, sms * w)
    if w <= 8:
        measure(f"k1d_w{w}_168regs", {"TFB_FORCE_KERNEL": "4", "TFB_K1D_W": str(w), "TFB_K1D_NOMID": "1"}, sms * w)
measure("k1e_wave", {"TFB_FORCE_KERNEL": "5"}, sms // 2)
for k in (100, 148, 200, 296, 400, 592, 800, 1024, 1184, 1500, 1776, 2048, 2500, 3000, 3552, 4096):
    measure(f"auto_{k}", {}, k, reps=3)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "k1d_warp_sweep.json"), "w"), indent=1)
