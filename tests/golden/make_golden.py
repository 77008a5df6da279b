"""Generate tests/golden/reference_vectors.npz by running the REFERENCE itself.

Run in the build container only (the reference is mounted read-only at
/root/reference and does not exist on the GPU box):

    python tests/golden/make_golden.py

Everything stored here is an output of the unmodified reference package
`encirc`; the tests compare our host layer, the oracle port and the GPU engine
against these arrays.
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import encirc  # noqa: E402
from encirc import (  # noqa: E402
    GateKind, LweParams, OracleBootstrapEngine, PoolConfig, ReferenceEngine, WorkerPool,
    add_bitwise, add_numberwise, decrypt_int, encrypt_int, keygen, mul_karatsuba, mul_naive,
)
from encirc.engine import TWO_INPUT_KINDS  # noqa: E402
from encirc.linalg import decrypt_matrix, encrypt_matrix, mat_mul_cannon, mat_mul_flat  # noqa: E402
from encirc.torus import lwe_linear, phase  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}
meta = {"numpy": np.__version__, "encirc": encirc.__version__}

params = LweParams()
key = keygen(params, seed=11)
out["key11_bits"] = key.bits.astype(np.uint8)
out["key2024_bits"] = keygen(params, seed=2024).bits.astype(np.uint8)


def words(sample):
    return np.concatenate([sample.a.astype(np.uint32), np.array([sample.b], dtype=np.uint32)])


# fresh encryptions: first 12 draws of engine seed 5 (bit pattern 1,0,1,1,0,0,...)
eng = OracleBootstrapEngine(key, seed=5)
bits = [1, 0, 1, 1, 0, 0, 1, 0, 1, 1, 1, 0]
fresh = [eng.encrypt(b) for b in bits]
out["enc5_bits"] = np.array(bits, dtype=np.uint8)
out["enc5_words"] = np.stack([words(c.sample) for c in fresh])
out["enc5_phase"] = np.array([phase(key, c.sample).word for c in fresh], dtype=np.uint32)

# gate linear forms on the first two fresh samples, all eight kinds
lin = []
for kind in TWO_INPUT_KINDS:
    cx, cy, off = encirc.engine._LINEAR[kind]
    lin.append(words(lwe_linear([fresh[0].sample, fresh[1].sample], [cx, cy], off * params.mu)))
out["linear_words"] = np.stack(lin)

# one launch of the reference's oracle engine: 8 kinds x 4 input combos (decrypted bits + words)
eng = OracleBootstrapEngine(key, seed=5)
xs = [eng.encrypt((i >> 1) & 1) for i in range(32)]
ys = [eng.encrypt(i & 1) for i in range(32)]
kinds = [TWO_INPUT_KINDS[i // 4] for i in range(32)]
batch = encirc.JobBatch(kinds, xs, ys)
outs = eng.pool.execute_batch(batch, eng)
out["launch_x_words"] = np.stack([words(c.sample) for c in xs])
out["launch_y_words"] = np.stack([words(c.sample) for c in ys])
out["launch_kind_ids"] = np.array([i // 4 for i in range(32)], dtype=np.uint8)
out["launch_out_words"] = np.stack([words(c.sample) for c in outs])
out["launch_out_bits"] = np.array([eng.decrypt(c) for c in outs], dtype=np.uint8)
# a second launch (600 NAND jobs -> 3 rng blocks) hashed, as test_engine.py:227-238 does
eng = OracleBootstrapEngine(key, seed=77, pool=WorkerPool(PoolConfig(workers=1)))
xs = [eng.encrypt(i % 2) for i in range(600)]
ys = [eng.encrypt((i // 2) % 2) for i in range(600)]
got = eng.eval_gate_batch(GateKind.NAND, xs, ys)
h = hashlib.sha256(b"".join(words(c.sample).tobytes() for c in got)).hexdigest()
meta["nand600_seed77_sha256"] = h

# circuit counts and results on the cleartext engine (data-independent counts)
rng = np.random.default_rng(123)
ref = ReferenceEngine(params, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 22)))
counts = {}
for n in (8, 16, 32):
    a, b = int(rng.integers(0, 1 << n, dtype=np.uint64)), int(rng.integers(0, 1 << n, dtype=np.uint64))
    for name, fn in (("add_bitwise", add_bitwise), ("add_numberwise", add_numberwise),
                     ("mul_naive", mul_naive), ("mul_karatsuba", mul_karatsuba)):
        x, y = encrypt_int(ref, a, n), encrypt_int(ref, b, n)
        ref.reset_stats()
        r = fn(x, y)
        counts[f"{name}_{n}"] = {"a": a, "b": b, "result": decrypt_int(ref, r), **ref.stats.as_record()}
for q in (2, 3, 4):
    A = rng.integers(0, 1 << 16, size=(q, q)).tolist()
    B = rng.integers(0, 1 << 16, size=(q, q)).tolist()
    for name, fn in (("mat_mul_flat", mat_mul_flat), ("mat_mul_cannon", mat_mul_cannon)):
        ea, eb = encrypt_matrix(ref, A, 16), encrypt_matrix(ref, B, 16)
        ref.reset_stats()
        c = fn(ea, eb)
        counts[f"{name}_{q}"] = {"A": A, "B": B, "result": decrypt_matrix(ref, c), **ref.stats.as_record()}
meta["circuits"] = counts
meta["margins"] = {k.value: ref.gate_margin(k) for k in TWO_INPUT_KINDS}
meta["fresh_bound"] = params.fresh_noise_bound

# wire formats (encirc/serialize.py): bytes produced by the reference
from encirc.linalg import encrypt_vector  # noqa: E402
from encirc.serialize import dump_int, dump_key, dump_matrix, dump_params, dump_sample, dump_vector  # noqa: E402

ser_eng = OracleBootstrapEngine(key, seed=9)
ser_int = encrypt_int(ser_eng, 11, 4)
ser_vec = encrypt_vector(ser_eng, [3, 5], 3)
ser_mat = encrypt_matrix(ser_eng, [[1, 2], [3, 0]], 2)
for name, blob in (("ser_params", dump_params(params)), ("ser_key11", dump_key(key)),
                   ("ser_sample", dump_sample(fresh[0].sample)), ("ser_int", dump_int(ser_int)),
                   ("ser_vector", dump_vector(ser_vec)), ("ser_matrix", dump_matrix(ser_mat))):
    out[name] = np.frombuffer(blob, dtype=np.uint8)

# rows of the reference's own harness on its cleartext engine, timing omitted (encirc/bench.py)
from encirc import bench as ref_bench  # noqa: E402

def harness_engine():
    return ReferenceEngine(params, pool=WorkerPool(PoolConfig(workers=1)), seed=3)

rows = []
rows += ref_bench.bench_gate(harness_engine(), (4, 8, 16, 32), (GateKind.AND, GateKind.XOR))
rows += ref_bench.bench_compound(harness_engine(), (1, 4, 8))
rows += ref_bench.bench_add(harness_engine(), (16, 32), "bitwise", (1, 4))
rows += ref_bench.bench_add(harness_engine(), (16,), "numberwise", (1,))
rows += ref_bench.bench_mul(harness_engine(), (16,), "naive", (1, 4))
rows += ref_bench.bench_mul(harness_engine(), (16,), "karatsuba", (1,))
rows += ref_bench.bench_matmul(harness_engine(), (2, 4), "cannon")
rows += ref_bench.bench_matmul(harness_engine(), (2,), "flat")
meta["harness_rows"] = [r.record(omit_timing=True) for r in rows]

# encrypted linear regression (encirc/regression.py, encirc/datasets.py) on the cleartext engine
from encirc import fit_encrypted, synthesize, to_csv_text  # noqa: E402

reg = {}
for kind in ("numerical", "binary"):
    ds = synthesize(kind, 12, 3, seed=4)
    eng_r = ReferenceEngine(params, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 22)))
    rep = fit_encrypted(eng_r, ds, bits=12)
    reg[kind] = {"csv": to_csv_text(ds), "truth": list(ds.coefficients),
                 "coefficients": [[c.numerator, c.denominator] for c in rep.coefficients],
                 "gram": [list(r) for r in rep.gram], "moment": list(rep.moment), "stats": eng_r.stats.as_record()}
meta["regression"] = reg

np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
with open(os.path.join(HERE, "reference_meta.json"), "w") as f:
    json.dump(meta, f, indent=1, sort_keys=True)
print("wrote", {k: v.shape for k, v in out.items()})
