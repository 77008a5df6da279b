"""First-light GPU script (not a pytest module): parity of every kernel against
the CPU oracle on a handful of gates, then a batch-size sweep.  Run under gpurun:
    python tests/gpu_first_light.py [--sweep] [--kmax 65536]
Writes gpurun_out/first_light.json."""
import argparse, ctypes, json, os, sys, time
import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_01945_b200 import _cabi
from paper_2005_01945_b200.keys import RingParams, generate_evaluation_keys
from paper_2005_01945_b200.torus import LweParams, encrypt_bit, keygen
from oracle import tfhe_oracle as orc

ap = argparse.ArgumentParser()
ap.add_argument("--sweep", action="store_true")
ap.add_argument("--kmax", type=int, default=65536)
ap.add_argument("--parity", type=int, default=16)
args = ap.parse_args()

dev = torch.device("cuda:0")
p = LweParams()
key = keygen(p, seed=11)
ek = generate_evaluation_keys(key, seed=11)
n = p.m
ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
t0 = time.time()
ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
report = {"load_keys_s": time.time() - t0}

# --- spectral key vs numpy ---
spec = np.empty((4, 2, 512, 2), dtype=np.float64)
ctx.call("tfb_debug_spectral_key", 7, spec.ctypes.data)
N = 1024
tw = np.exp(1j * np.pi * np.arange(N // 2) / N)
poly = ek.bk[7].astype(np.float64)  # [4][2][N]
z = (poly[..., : N // 2] + 1j * poly[..., N // 2 :]) * tw
want = np.fft.ifft(z, axis=-1) * (N // 2)
got = spec[..., 0] + 1j * spec[..., 1]
report["spectral_key_rel_err"] = float(np.abs(got - want).max() / np.abs(want).max())

# --- parity on a few gates ---
rng = np.random.default_rng((11, 0))
def pack(s):
    return np.concatenate([s.a, [s.b]]).astype(np.uint32)
K = args.parity
xs = np.stack([pack(encrypt_bit(key, (g >> 1) & 1, rng)) for g in range(K)])
ys = np.stack([pack(encrypt_bit(key, g & 1, rng)) for g in range(K)])
kinds = np.array([(g // 4) % 8 for g in range(K)], dtype=np.uint8)
want_out, want_ext = orc.gate_bootstrap_batch(xs, ys, kinds, p.mu.word, ek.bk, ek.ksk, want_ext=True)

pool = torch.zeros((3 * K, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
pool[:K, : n + 1] = torch.from_numpy(xs.view(np.int32)).to(dev)
pool[K : 2 * K, : n + 1] = torch.from_numpy(ys.view(np.int32)).to(dev)
kinds_d = torch.from_numpy(kinds).to(dev)
xr = torch.arange(0, K, dtype=torch.int32, device=dev)
yr = torch.arange(K, 2 * K, dtype=torch.int32, device=dev)
orow = torch.arange(2 * K, 3 * K, dtype=torch.int32, device=dev)
ext = torch.zeros((K, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)
ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kinds_d.data_ptr(), xr.data_ptr(), yr.data_ptr(), ext.data_ptr(), K, None)
torch.cuda.synchronize()
got_ext = ext.cpu().numpy().view(np.uint32)[:, : N + 1]
report["blind_rotate_mismatch_words"] = int((got_ext != want_ext).sum())
ctx.call("tfb_gate_launch", pool.data_ptr(), kinds_d.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow.data_ptr(), K, None)
torch.cuda.synchronize()
got_out = pool[2 * K :, : n + 1].cpu().numpy().view(np.uint32)
report["gate_mismatch_words"] = int((got_out != want_out).sum())
# host-buffer path
out_h = np.zeros((K, n + 1), dtype=np.uint32)
ctx.call("tfb_gate_launch_host", xs.ctypes.data, ys.ctypes.data, kinds.ctypes.data, out_h.ctypes.data, K)
report["host_path_mismatch_words"] = int((out_h != want_out).sum())
# decrypt
TT = {0: (0, 0, 0, 1), 1: (0, 1, 1, 1), 2: (1, 1, 1, 0), 3: (1, 0, 0, 0), 4: (0, 1, 1, 0), 5: (1, 0, 0, 1), 6: (0, 1, 0, 0), 7: (1, 1, 0, 1)}
bad = 0
for g in range(K):
    ph = orc.lwe_phase(got_out[g], key.bits)
    bit = 1 if 0 < ph < 2**31 else 0
    bad += bit != TT[int(kinds[g])][(((g >> 1) & 1) << 1) | (g & 1)]
report["decrypt_errors"] = int(bad)
print(json.dumps(report), flush=True)

# --- peaks ---
report["peaks"] = _cabi.measure_peaks(0)
print(report["peaks"], flush=True)

# --- sweep ---
if args.sweep:
    sweep = []
    k = 1
    ks = []
    while k <= args.kmax:
        ks.append(k); k *= 4
    for k in sorted(set(ks + [148 * 4, 148 * 16, args.kmax])):
        if k > args.kmax: continue
        pool = torch.zeros((3 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
        src = torch.from_numpy(xs.view(np.int32)).to(dev)
        idx = torch.arange(k, device=dev) % K
        pool[:k, : n + 1] = src[idx]
        pool[k : 2 * k, : n + 1] = torch.from_numpy(ys.view(np.int32)).to(dev)[idx]
        kd = kinds_d[idx].contiguous()
        xr = torch.arange(0, k, dtype=torch.int32, device=dev)
        yr = torch.arange(k, 2 * k, dtype=torch.int32, device=dev)
        orow = torch.arange(2 * k, 3 * k, dtype=torch.int32, device=dev)
        ext = torch.zeros((k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)
        def run_full():
            ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow.data_ptr(), k, None)
        def run_br():
            ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kd.data_ptr(), xr.data_ptr(), yr.data_ptr(), ext.data_ptr(), k, None)
        def run_ks():
            ctx.call("tfb_debug_key_switch", ext.data_ptr(), pool.data_ptr(), orow.data_ptr(), k, None)
        row = {"k": k}
        for name, fn in (("full", run_full), ("blind_rotate", run_br), ("key_switch", run_ks)):
            fn(); torch.cuda.synchronize()
            reps = 3 if k <= 4096 else 1
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps): fn()
            e1.record(); torch.cuda.synchronize()
            row[name + "_ms"] = e0.elapsed_time(e1) / reps
        row["gates_per_s"] = k / (row["full_ms"] * 1e-3)
        got = pool[2 * k : 2 * k + K, : n + 1].cpu().numpy().view(np.uint32)
        row["parity_ok"] = bool((got == want_out[: min(K, k)]).all()) if k >= K else bool((got[:k] == want_out[:k]).all())
        sweep.append(row)
        print(row, flush=True)
    report["sweep"] = sweep

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "first_light.json"), "w") as f:
    json.dump(report, f, indent=1)
print("DONE", json.dumps({k: v for k, v in report.items() if k != "sweep"}))
