"""Empirical output-noise statistics of the GPU bootstrap: phase error of gate
outputs against +-mu over many gates, for the two noisiest gate shapes.
    python tools/noise_stats.py [--gates 1048576] [--out gpurun_out/noise.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_01945_b200 import B200Engine, GateKind, LweParams, PoolConfig, WorkerPool, keygen, truth_table  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gates", type=int, default=1 << 20)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "noise.json"))
args = ap.parse_args()
key = keygen(LweParams(), seed=2024)
eng = B200Engine(key, seed=42, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 18)))
rng = np.random.default_rng(7)
base = 4096
bits = rng.integers(0, 2, size=base)
rows0, own0 = eng.encrypt_rows(bits.tolist())
report = {"gates_per_kind": args.gates, "fresh_bound": eng.fresh_bound}
for kind in (GateKind.NAND, GateKind.XOR):
    tt = np.array(truth_table(kind))
    # level 1: fresh inputs; level 2: inputs that are themselves bootstrapped outputs
    for level in (1, 2):
        errs = []
        done = 0
        while done < args.gates:
            k = min(1 << 18, args.gates - done)
            i, j = rng.integers(0, base, size=k), rng.integers(0, base, size=k)
            if level == 1:
                xr, yr, bx, by = rows0[i], rows0[j], bits[i], bits[j]
            else:
                mid, own_mid = eng.gate_rows(GateKind.NAND, rows0[i], rows0[j])
                bm = 1 - (bits[i] & bits[j])
                xr, yr, bx, by = mid, np.roll(mid, 1), bm, np.roll(bm, 1)
            out, own = eng.gate_rows(kind, xr, yr)
            want = tt[(bx << 1) | by]
            ph = eng.phases(out).astype(np.int64)
            target = np.where(want == 1, 1 << 29, (1 << 32) - (1 << 29))
            e = (((ph - target + 2**31) % 2**32) - 2**31) / 2.0**32
            assert np.array_equal(((ph > 0) & (ph < 2**31)).astype(int), want)
            errs.append(e)
            done += k
        e = np.concatenate(errs)
        report[f"{kind.value}_level{level}"] = {
            "std": float(e.std()), "max_abs": float(np.abs(e).max()), "mean": float(e.mean()),
            "exceed_fresh_bound": int((np.abs(e) >= eng.fresh_bound).sum()),
            "sigmas_to_bound": float(eng.fresh_bound / e.std()),
            "count": int(e.size),
            # tail counts against the Gaussian prediction 2 Q(z) * count (the bound sits at ~6.4 sigma)
            "tail_counts": {f"{z}": int((np.abs(e - e.mean()) > z * e.std()).sum()) for z in (4.0, 4.5, 5.0, 5.5, 6.0)},
        }
        print(kind.value, level, report[f"{kind.value}_level{level}"], flush=True)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(report, open(args.out, "w"), indent=1)
