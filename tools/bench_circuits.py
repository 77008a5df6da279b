"""Circuit-level timings on one B200 through the public engine API
(BASELINE.json configs 0, 2, 3, 4): single-gate latency, batch sweep, 16/32-bit
add and multiply, vector add / multiply and matrix products, every result
decrypted and compared with native integer arithmetic (as encirc/bench.py does).

    python tools/bench_circuits.py [--full] [--out gpurun_out/circuits.json]

--full adds the two largest workloads (vec_mul 4096 x 32-bit: 44.8 M bootstraps;
16 x 16 Cannon matmul at 16 bits: 11.5 M bootstraps).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_01945_b200 import (  # noqa: E402
    B200Engine, GateKind, LweParams, PoolConfig, WorkerPool, add_bitwise, add_numberwise, decrypt_int,
    decrypt_matrix, decrypt_vector, encrypt_int, encrypt_matrix, encrypt_vector, keygen, mat_mul_cannon,
    mat_mul_flat, mul_karatsuba, mul_naive, truth_table, vec_add, vec_mul,
)

ap = argparse.ArgumentParser()
ap.add_argument("--full", action="store_true")
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "circuits.json"))
args = ap.parse_args()

key = keygen(LweParams(), seed=2024)
eng = B200Engine(key, seed=42, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 23)),
                 initial_rows=1 << 18)  # 512 MB of rows up front: pool growth (a cudaMalloc) stays out of the timed regions
rng = np.random.default_rng((42, 2))
rows = []


def timed(name, fn, check, **extra):
    eng.synchronize()
    eng.reset_stats()
    t0 = time.perf_counter()
    out = fn()
    eng.synchronize()
    dt = time.perf_counter() - t0
    st = eng.stats.as_record()
    ok = bool(check(out))
    rec = {"experiment": name, "seconds": dt, "correct": ok, **st, **extra}
    if st["bootstraps"]:
        rec["gates_per_s"] = st["bootstraps"] / dt
    rows.append(rec)
    print(json.dumps(rec), flush=True)
    return out


# config 0: single-gate latency (sequential dependent calls)
x, y = eng.encrypt(1), eng.encrypt(0)
for kind in (GateKind.NAND, GateKind.AND, GateKind.XOR):
    eng.eval_gate(kind, x, y)
    eng.synchronize()
    lat = []
    for _ in range(200):
        t0 = time.perf_counter()
        out = eng.eval_gate(kind, x, y)
        eng.synchronize()
        lat.append(time.perf_counter() - t0)
    rec = {"experiment": f"single-gate-{kind.value.lower()}", "median_us": float(np.median(lat)) * 1e6,
           "p10_us": float(np.percentile(lat, 10)) * 1e6, "correct": eng.decrypt(out) == truth_table(kind)[2]}
    rows.append(rec)
    print(json.dumps(rec), flush=True)

# config 1: batch sweep through the engine API (index arrays), includes host overhead
for k in (1, 16, 256, 1024, 4096, 16384, 65536):
    bits = rng.integers(0, 2, size=(2, k))
    xr, xo = eng.encrypt_rows(bits[0].tolist())
    yr, yo = eng.encrypt_rows(bits[1].tolist())
    eng.gate_rows(GateKind.NAND, xr, yr)
    timed(f"gate-batch-nand-{k}", lambda: eng.gate_rows(GateKind.NAND, xr, yr),
          lambda o: np.array_equal(eng.decrypt_rows(o[0]), 1 - (bits[0] & bits[1])), k=k)
    if k >= 1024:
        timed(f"compound-xor-and-{k}", lambda: eng.compound_rows(GateKind.XOR, GateKind.AND, xr, yr),
              lambda o: np.array_equal(eng.decrypt_rows(o[0]), bits[0] ^ bits[1])
              and np.array_equal(eng.decrypt_rows(o[1]), bits[0] & bits[1]), k=k)
    del xr, yr, xo, yo

# configs 2, 3: scalar add / multiply
for n in (16, 32):
    a, b = int(rng.integers(0, 1 << n, dtype=np.uint64)), int(rng.integers(0, 1 << n, dtype=np.uint64))
    ex, ey = encrypt_int(eng, a, n), encrypt_int(eng, b, n)
    timed(f"add-bitwise-{n}", lambda: add_bitwise(ex, ey), lambda r: decrypt_int(eng, r) == (a + b) % (1 << n), n=n)
    timed(f"add-numberwise-{n}", lambda: add_numberwise(ex, ey), lambda r: decrypt_int(eng, r) == (a + b) % (1 << n), n=n)
    timed(f"mul-naive-{n}", lambda: mul_naive(ex, ey), lambda r: decrypt_int(eng, r) == a * b, n=n)
    timed(f"mul-karatsuba-{n}", lambda: mul_karatsuba(ex, ey), lambda r: decrypt_int(eng, r) == a * b, n=n)

# config 4: vectors and matrices
def vec_case(ell, n, mul):
    u = rng.integers(0, 1 << n, size=ell, dtype=np.uint64).tolist()
    v = rng.integers(0, 1 << n, size=ell, dtype=np.uint64).tolist()
    t0 = time.perf_counter()
    eu, ev = encrypt_vector(eng, u, n), encrypt_vector(eng, v, n)
    enc_s = time.perf_counter() - t0
    if mul:
        timed(f"vec-mul-{ell}x{n}", lambda: vec_mul(eu, ev),
              lambda r: decrypt_vector(eng, r) == [int(a) * int(b) for a, b in zip(u, v)], n=n, ell=ell, encrypt_seconds=enc_s)
    else:
        timed(f"vec-add-{ell}x{n}", lambda: vec_add(eu, ev),
              lambda r: decrypt_vector(eng, r) == [(int(a) + int(b)) % (1 << n) for a, b in zip(u, v)], n=n, ell=ell,
              encrypt_seconds=enc_s)


vec_case(32, 32, False)
vec_case(4096, 32, False)
vec_case(32, 32, True)
if args.full:
    vec_case(4096, 32, True)


def mat_case(q, n, fn, name):
    A = rng.integers(0, 1 << n, size=(q, q)).tolist()
    B = rng.integers(0, 1 << n, size=(q, q)).tolist()
    want = [[sum(A[i][t] * B[t][j] for t in range(q)) % (1 << n) for j in range(q)] for i in range(q)]
    ea, eb = encrypt_matrix(eng, A, n), encrypt_matrix(eng, B, n)
    timed(f"{name}-{q}x{q}-{n}", lambda: fn(ea, eb), lambda r: decrypt_matrix(eng, r) == want, n=n, rank=q)


mat_case(4, 16, mat_mul_cannon, "matmul-cannon")
mat_case(4, 16, mat_mul_flat, "matmul-flat")
mat_case(8, 16, mat_mul_cannon, "matmul-cannon")
if args.full:
    mat_case(16, 16, mat_mul_cannon, "matmul-cannon")
    mat_case(16, 16, lambda a, b: mat_mul_flat(a, b, max_jobs=1 << 24), "matmul-flat")

os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    json.dump({"device": "B200", "kernel_launches": eng.kernel_launches, "rows": rows}, f, indent=1)
print("wrote", args.out)
