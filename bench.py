"""bench.py -- bootstrapped gates/sec on B200 and 32-bit encrypted add / mul ops/sec vs the CPU reference
(BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload gates|vec_add|vec_mul|matmul16] [--batch 65536]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N ... bench.py --gpus N ...

Default workload `gates` (BASELINE configs[1]): a step is one launch of `batch` = 2**16 independent
bootstrapped NAND gates at the reference's default parameter set, synthetic random plaintexts, inputs resident
in HBM.  `value` is whole-job gates/s over N GPUs, weak scaling (every rank runs its own launch; gates are
independent: no data-path collective, NCCL broadcasts the evaluation keys and reduces timings / checks).
`e2e` is the same metric through the C ABI's host-buffer entry point, host<->device copies inside the timed
region.  `roofline` is the fused bootstrap kernel against the FP64 pipe (bound by transform + MAC
FP64 work, not HBM, not tensor cores), DFMA peak measured in the same run.

Workloads `vec_add` / `vec_mul` / `matmul16` (BASELINE configs[4]) are the sharded circuits of
paper_2005_01945_b200/sharding.py at full size (4096 x 32-bit vectors, 16 x 16 matrix of 16-bit cells): strong
scaling, a step is one whole operation (scatter / broadcast of the operand ciphertexts, the circuit on every
rank's block, gather of the result), `value` = logical bootstraps of the operation / time.  The default line
also carries `sharded.vec_add` so that every N reports one strong-scaling figure.

At N = 1 the line also carries: `cpu_baseline` (the reference's own engine from oracle/_ref, workers = 1 and
all cores, on a bounded sample), `cpu_real_bootstrap` (our C restatement of the REAL bootstrap: the like-for-like
CPU comparator; the reference's "bootstrap" is a decrypt / re-encrypt oracle), `circuits` (16/32-bit add and
multiply on the GPU and, timed in the same run, on the reference's CPU engine), `latency` (configs[0]: median
over 1,000 sequential single gates per kind) and `sweep` (configs[1]: gates/s against launch size).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "bootstrapped_gates_per_sec"
UNIT = "gates/s"
KEY_SEED, ENGINE_SEED = 2024, 42
NAND = 2
# Algorithmic FP64 work of one gate with the bootstrapping key unrolled over pairs of mask elements (SURVEY 8(d)'s count
# restated for 250 pair steps instead of 500 CMux steps): per step 6 negacyclic transforms of 26,112 FLOP (radix-2 count
# incl. the twist) and, per spectral point (512) and digit polynomial (4), the key combination K = u1 B1 + u2 B2 + u1 u2 B12
# for both output components (2 x 3 complex multiply-adds = 48 FLOP) and the two MACs (16 FLOP), plus the two rotation
# factors once per point (14 FLOP): 156,672 + 512 x (4 x 64 + 14) = 294,912 FLOP per step, 73.73 MFLOP per gate.
# (The plain CMux loop of round 1 was 500 x (6 x 26,112 + 32,768) = 94.72 MFLOP per gate.)
FLOP_PER_GATE = 250 * (6 * 26112 + 512 * (4 * 64 + 14))
FLOP_PER_GATE_PLAIN_CMUX = 500 * (6 * 26112 + 32768)
SHARDED = {"vec_add": (4096, 32), "vec_mul": (4096, 32), "matmul16": (16, 16)}  # (lanes | rank, bit width)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="gates", choices=["gates", *SHARDED])
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--lanes", type=int, default=None, help="override the lane count / matrix rank of a sharded workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-circuits", action="store_true")
    ap.add_argument("--no-sharded", action="store_true")
    return ap.parse_args()


def config(args, n_gpus):
    cfg = {
        "params": "m=500 alpha=2^-15 w=32 mu=1/8; ring N=1024 k=1 l=2 Bg=2^9 ks t=8 base=4; bootstrapping key unrolled over pairs of mask elements (250 blind-rotation steps)",
    }
    if args.workload == "gates":
        cfg.update({
            "workload": "BASELINE configs[1]: batched independent NAND gates, one launch per step",
            "batch_per_gpu": args.batch,
            "parallelism": f"gates sharded over {n_gpus} GPU(s), no data-path collective",
            "l2": "inputs (2 x batch x 2 KiB = 268 MB) exceed the 126 MB L2; no flush needed",
        })
    else:
        lanes, width = sharded_shape(args)
        what = (f"16x16-class matrix product, rank {lanes}, {width}-bit cells, output cells sharded (flat per-cell schedule)"
                if args.workload == "matmul16" else f"{args.workload} of {lanes} x {width}-bit lanes, lanes sharded")
        cfg.update({
            "workload": f"BASELINE configs[4]: {what}; one whole operation per step incl. scatter/gather",
            "parallelism": f"strong scaling over {n_gpus} GPU(s); NCCL scatter/broadcast of operands, gather of results",
            "l2": "operand + intermediate ciphertexts (>= 0.5 GB) exceed the 126 MB L2; no flush needed",
        })
    return cfg


def sharded_shape(args):
    lanes, width = SHARDED[args.workload]
    return (args.lanes or lanes), width


def synth_inputs(key_bits: np.ndarray, k: int, seed: int):
    """Vectorised fresh encryptions of uniform random bits (same distribution as encirc/torus.py:254-271; the
    draw order differs, which only matters to the parity tests, not to throughput)."""
    rng = np.random.default_rng((seed, 2))
    bits = rng.integers(0, 2, size=(2, k))
    words = np.empty((2, k, len(key_bits) + 1), dtype=np.uint32)
    words[:, :, :-1] = rng.integers(0, 1 << 32, size=(2, k, len(key_bits)), dtype=np.uint32)
    noise = np.clip(np.rint(rng.normal(0.0, 2.0**-15, size=(2, k)) * 2.0**32), -(2**27 - 1), 2**27 - 1)
    msg = np.where(bits == 1, 1 << 29, (1 << 32) - (1 << 29))
    body = (words[:, :, :-1] @ key_bits.astype(np.uint32)).astype(np.int64) + msg + noise.astype(np.int64)
    words[:, :, -1] = (body % (1 << 32)).astype(np.uint32)
    return bits, words


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, smax, reasons, power = [], [], set(), []
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax.append(float(f[2])); power.append(float(f[3]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [c for c, p in zip(sm, power) if p > 0.5 * max(power)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "power_w_max": max(power), "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref: the unmodified reference staged by oracle/make_ref.py;
# oracle/encirc_port.py, pinned bit-exactly to it, only where the staged copy is absent)
# ------------------------------------------------------------------------------------------

def load_reference():
    try:
        from oracle.make_ref import import_reference

        return import_reference()
    except ImportError:
        return None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def time_reference_gates(encirc, k: int, steps: int, warmup: int, workers: int):
    """The reference's own engine on `k` NAND gates per step in one launch (max_batch = k), encryption outside
    the timed region like encirc/bench.py:179-190.  Returns (gates/s, s/step, outputs verified)."""
    key = encirc.keygen(encirc.LweParams(), seed=KEY_SEED)
    pool = encirc.WorkerPool(encirc.PoolConfig(workers=workers, max_batch=k))
    eng = encirc.OracleBootstrapEngine(key, seed=ENGINE_SEED, pool=pool)
    bits, words = synth_inputs(np.asarray(key.bits), k, ENGINE_SEED)
    fresh, w = key.params.fresh_noise_bound, key.params.w
    xs = [encirc.EncBit(eng, sample=encirc.LweSample(words[0, i, :-1], int(words[0, i, -1]), fresh, w)) for i in range(k)]
    ys = [encirc.EncBit(eng, sample=encirc.LweSample(words[1, i, :-1], int(words[1, i, -1]), fresh, w)) for i in range(k)]
    for _ in range(warmup):
        outs = eng.eval_gate_batch(encirc.GateKind.NAND, xs, ys)
    t0 = time.perf_counter()
    for _ in range(steps):
        outs = eng.eval_gate_batch(encirc.GateKind.NAND, xs, ys)
    dt = time.perf_counter() - t0
    got = np.array([eng.decrypt(c) for c in outs[:2048]])
    ok = bool(np.array_equal(got, 1 - (bits[0, :2048] & bits[1, :2048])))
    pool.shutdown()
    return k * steps / dt, dt / steps, ok


def time_port_gates(k: int, steps: int, warmup: int):
    from oracle import encirc_port as port

    key_bits = port.keygen_bits(KEY_SEED)
    eng = port.OracleLweEngine(key_bits, seed=ENGINE_SEED, max_batch=k)
    bits, words = synth_inputs(key_bits, k, ENGINE_SEED)
    xs = [port.Sample(words[0, i, :-1], words[0, i, -1], port.FRESH_BOUND) for i in range(k)]
    ys = [port.Sample(words[1, i, :-1], words[1, i, -1], port.FRESH_BOUND) for i in range(k)]
    for _ in range(warmup):
        outs = eng.eval_gate_batch(NAND, xs, ys)
    t0 = time.perf_counter()
    for _ in range(steps):
        outs = eng.eval_gate_batch(NAND, xs, ys)
    dt = time.perf_counter() - t0
    got = np.array([eng.decrypt(c) for c in outs[:2048]])
    return k * steps / dt, dt / steps, bool(np.array_equal(got, 1 - (bits[0, :2048] & bits[1, :2048])))


def reference_gate_rates(k: int, steps: int, warmup: int) -> dict:
    """cpu_baseline record: the reference at workers = 1 and workers = all cores; `value` is the
    better of the two."""
    encirc = load_reference()
    cores = host_cores()
    if encirc is None:
        v, per, ok = time_port_gates(k, steps, warmup)
        return {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "correct": ok, "s_per_step": per,
                "sample": f"{k} NAND gates per launch, {steps} timed launches; oracle/encirc_port.py (oracle/_ref not staged)"}
    runs = {}
    for workers in sorted({1, cores}):
        v, per, ok = time_reference_gates(encirc, k, steps, warmup, workers)
        runs[workers] = {"gates_per_s": v, "s_per_step": per, "correct": ok}
    best = max(runs, key=lambda wk: runs[wk]["gates_per_s"])
    return {"value": runs[best]["gates_per_s"], "unit": UNIT, "cores": best, "kind": "reference",
            "host_cores": cores, "s_per_step": runs[best]["s_per_step"],
            "correct": all(r["correct"] for r in runs.values()),
            "by_workers": {str(wk): r for wk, r in runs.items()},
            "sample": f"{k} NAND gates per launch, {steps} timed launches; the unmodified reference "
                      "(oracle/_ref: encirc.OracleBootstrapEngine.eval_gate_batch, max_batch = launch size)"}


def reference_circuit_seconds(workers_list=None) -> dict | None:
    """add_bitwise / mul_naive at 16 and 32 bits on the reference's own engine (encirc/integers.py:116-120,
    241-244), best of 3, per worker count; plus the batched forms used for the ops/sec throughput figure."""
    encirc = load_reference()
    if encirc is None:
        return None
    key = encirc.keygen(encirc.LweParams(), seed=KEY_SEED)
    rng = np.random.default_rng((ENGINE_SEED, 2))
    out = {"host_cores": host_cores(), "kind": "reference"}
    for workers in (workers_list or sorted({1, host_cores()})):
        pool = encirc.WorkerPool(encirc.PoolConfig(workers=workers, max_batch=1 << 16))
        eng = encirc.OracleBootstrapEngine(key, seed=ENGINE_SEED, pool=pool)
        rec = {}
        for n in (16, 32):
            a, b = (int(v) for v in rng.integers(0, 1 << n, size=2, dtype=np.uint64))
            x, y = encirc.encrypt_int(eng, a, n), encirc.encrypt_int(eng, b, n)
            for name, fn, want in ((f"add{n}", encirc.add_bitwise, (a + b) % (1 << n)), (f"mul{n}", encirc.mul_naive, a * b),
                                   (f"karatsuba{n}", encirc.mul_karatsuba, a * b)):
                best = None
                for _ in range(3):
                    t0 = time.perf_counter()
                    res = fn(x, y)
                    dt = time.perf_counter() - t0
                    best = dt if best is None else min(best, dt)
                rec[name] = {"seconds": best, "correct": encirc.decrypt_int(eng, res) == want}
        for name, lanes, fn in (("add32_x256", 256, encirc.vec_add), ("mul32_x16", 16, encirc.vec_mul)):
            u = [int(v) for v in rng.integers(0, 1 << 32, size=lanes, dtype=np.uint64)]
            v = [int(v) for v in rng.integers(0, 1 << 32, size=lanes, dtype=np.uint64)]
            U, V = encirc.encrypt_vector(eng, u, 32), encirc.encrypt_vector(eng, v, 32)
            t0 = time.perf_counter()
            res = fn(U, V)
            dt = time.perf_counter() - t0
            want = [(p + q) % (1 << 32) for p, q in zip(u, v)] if fn is encirc.vec_add else [p * q for p, q in zip(u, v)]
            rec[name] = {"seconds": dt, "ops_per_s": lanes / dt, "correct": encirc.decrypt_vector(eng, res) == want}
        out[f"workers_{workers}"] = rec
        pool.shutdown()
    return out


def time_real_bootstrap_cpu(sample: int):
    """Our C restatement of the real TFHE bootstrap (double-precision FFT path), all host threads: the
    like-for-like CPU comparator."""
    from oracle import tfhe_oracle as orc
    from paper_2005_01945_b200 import LweParams, generate_evaluation_keys, keygen

    key = keygen(LweParams(), seed=KEY_SEED)
    ek = generate_evaluation_keys(key, seed=ENGINE_SEED)
    bits, words = synth_inputs(key.bits, sample, ENGINE_SEED)
    kinds = np.full(sample, NAND, dtype=np.uint8)
    orc.gate_bootstrap_batch(words[0, :8], words[1, :8], kinds[:8], key.params.mu.word, ek.bk, ek.ksk, fft=True)
    t0 = time.perf_counter()
    out = orc.gate_bootstrap_batch(words[0], words[1], kinds, key.params.mu.word, ek.bk, ek.ksk, fft=True)
    dt = time.perf_counter() - t0
    ph = (out[:, -1].astype(np.int64) - (out[:, :-1] @ key.bits.astype(np.uint32)).astype(np.int64)) % (1 << 32)
    ok = bool(np.array_equal(((ph > 0) & (ph < 2**31)).astype(int), 1 - (bits[0] & bits[1])))
    return sample / dt, orc.max_threads(), ok


def reference_sharded_sample(args) -> tuple:
    """The reference's vec_add / vec_mul / mat_mul_flat on a bounded slice of the workload (lanes are independent
    and the cost is linear in them: SURVEY 6.3): (bootstraps/s, seconds, sample text, verified, cores)."""
    encirc = load_reference()
    if encirc is None:
        raise SystemExit(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not staged; the port has no circuits"}))
    lanes, width = sharded_shape(args)
    cores = host_cores()
    key = encirc.keygen(encirc.LweParams(), seed=KEY_SEED)
    rng = np.random.default_rng((ENGINE_SEED, 2))
    best = None
    for workers in sorted({1, cores}):
        pool = encirc.WorkerPool(encirc.PoolConfig(workers=workers, max_batch=1 << 16))
        eng = encirc.OracleBootstrapEngine(key, seed=ENGINE_SEED, pool=pool)
        if args.workload == "matmul16":
            q = min(lanes, 4)
            a, b = (rng.integers(0, 1 << width, size=(q, q)).tolist() for _ in range(2))
            A, B = encirc.encrypt_matrix(eng, a, width), encirc.encrypt_matrix(eng, b, width)
            eng.reset_stats()
            t0 = time.perf_counter()
            res = encirc.mat_mul_flat(A, B)
            dt = time.perf_counter() - t0
            ok = encirc.decrypt_matrix(eng, res) == [[sum(a[i][t] * b[t][j] for t in range(q)) % (1 << width)
                                                      for j in range(q)] for i in range(q)]
            text = f"mat_mul_flat rank {q} (of {lanes}), {width}-bit"
        else:
            ell = min(lanes, 256 if args.workload == "vec_add" else 16)
            u = [int(v) for v in rng.integers(0, 1 << width, size=ell, dtype=np.uint64)]
            v = [int(v) for v in rng.integers(0, 1 << width, size=ell, dtype=np.uint64)]
            U, V = encirc.encrypt_vector(eng, u, width), encirc.encrypt_vector(eng, v, width)
            fn = encirc.vec_add if args.workload == "vec_add" else encirc.vec_mul
            eng.reset_stats()
            t0 = time.perf_counter()
            res = fn(U, V)
            dt = time.perf_counter() - t0
            want = [(p + q_) % (1 << width) for p, q_ in zip(u, v)] if fn is encirc.vec_add else [p * q_ for p, q_ in zip(u, v)]
            ok = encirc.decrypt_vector(eng, res) == want
            text = f"{args.workload} of {ell} (of {lanes}) x {width}-bit lanes"
        rate = eng.stats.bootstraps / dt
        pool.shutdown()
        if best is None or rate > best[0]:
            best = (rate, dt, text + f", workers={workers}", ok, workers)
    return best


def run_reference(args) -> None:
    """The reference's own CPU implementation of the path on the box's host cores (rank 0 only)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if args.workload == "gates":
        k = min(args.batch, 1 << 16)
        base = reference_gate_rates(k, max(1, args.steps), max(1, min(args.warmup, 2)))
        value, per_step, ok, cores = base["value"], base["s_per_step"], base["correct"], base["cores"]
    else:
        value, per_step, text, ok, cores = reference_sharded_sample(args)
        base = {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "host_cores": host_cores(), "sample": text}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.workload == "gates" else "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": config(args, args.gpus), "cpu_baseline": base,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "correct": ok,
        "note": "the reference CPU path is a key-holding oracle (one 500-long dot product + RNG per gate), not a TFHE bootstrap",
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------

class Job:
    """One rank of the B200 arm: engine, NCCL plumbing, timing helpers."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        from paper_2005_01945_b200 import B200Engine, LweParams, PoolConfig, WorkerPool, _cabi, keygen
        from paper_2005_01945_b200.sharding import broadcast_eval_keys

        self.args, self.torch, self.dist, self._cabi = args, torch, dist, _cabi
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.distributed = "RANK" in os.environ and "WORLD_SIZE" in os.environ  # launched by torch.distributed.run
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.distributed:
            dist.init_process_group("nccl", device_id=self.dev)
        self.key = keygen(LweParams(), seed=KEY_SEED)
        # evaluation keys: generated on rank 0, broadcast raw over NCCL, transformed on every GPU (kernel K3)
        raw = broadcast_eval_keys(self.key, ENGINE_SEED, self.dev)
        self.eng = B200Engine(self.key, seed=ENGINE_SEED + self.rank, device=self.local, raw_key_tensors=raw,
                              device_encrypt=True, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 22)))
        del raw
        self.ctx = self.eng._ctx
        self.stream = torch.cuda.current_stream(self.dev).cuda_stream

    def fence(self):
        if self.distributed:
            self.dist.barrier()
        self.torch.cuda.synchronize(self.dev)

    def timed(self, fn, reps) -> float:
        """ms for `reps` calls: CUDA events on the launching stream, barrier + synchronize on both sides, MAX over ranks."""
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.fence()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        self.fence()
        return self.max_over_ranks(e0.elapsed_time(e1))

    def max_over_ranks(self, x: float) -> float:
        if not self.distributed:
            return float(x)
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_true(self, flag: bool) -> bool:
        if not self.distributed:
            return bool(flag)
        t = self.torch.tensor([int(flag)], device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return bool(t.item())

    def close(self):
        if self.distributed:
            self.dist.destroy_process_group()


def gates_workload(job: Job) -> dict:
    """configs[1]: one launch of `batch` NAND gates per step and rank; value, K1-only roofline, e2e."""
    torch, ctx, dev, args, _cabi = job.torch, job.ctx, job.dev, job.args, job._cabi
    n, k = job.key.params.m, args.batch
    bits, words = synth_inputs(job.key.bits, k, ENGINE_SEED + job.rank)
    pool = torch.zeros((3 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
    pool[:k, : n + 1] = torch.from_numpy(words[0].view(np.int32)).to(dev)
    pool[k : 2 * k, : n + 1] = torch.from_numpy(words[1].view(np.int32)).to(dev)
    kinds = torch.full((k,), NAND, dtype=torch.uint8, device=dev)
    idx = torch.arange(3 * k, dtype=torch.int32, device=dev)
    xr, yr, orow = idx[:k], idx[k : 2 * k], idx[2 * k :]
    key_bits_t = torch.from_numpy(job.key.bits.astype(np.uint32).view(np.int32)).to(dev)

    def step():
        ctx.call("tfb_gate_launch", pool.data_ptr(), kinds.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow.data_ptr(),
                 k, job.stream)

    for _ in range(args.warmup):
        step()
    launches0 = ctx.kernel_launches
    with ClockSampler(job.local) as clocks:
        total_ms = job.timed(step, args.steps)
    gpu_launches = ctx.kernel_launches - launches0
    value = job.world * k * args.steps / (total_ms * 1e-3)

    # correctness of the timed work: every output of the last step decrypts to NAND
    ph = torch.empty(k, dtype=torch.int32, device=dev)
    ctx.call("tfb_rows_phase", pool.data_ptr(), orow.data_ptr(), key_bits_t.data_ptr(), ph.data_ptr(), k, job.stream)
    phase = ph.cpu().numpy().view(np.uint32)
    correct = job.all_true(np.array_equal(((phase > 0) & (phase < 2**31)).astype(int), 1 - (bits[0] & bits[1])))

    # launch-size sweep (configs[1]): gates/s against k, same pool prefix
    sweep = {}
    if job.rank == 0 and job.world == 1:
        for kk in [1 << e for e in range(0, 17)]:
            kk = min(kk, k)

            def part(kk=kk):
                ctx.call("tfb_gate_launch", pool.data_ptr(), kinds.data_ptr(), xr.data_ptr(), yr.data_ptr(),
                         orow.data_ptr(), kk, job.stream)

            part()
            reps = 3 if kk >= 4096 else 10
            sweep[str(kk)] = kk * reps / (job.timed(part, reps) * 1e-3)

    # configs[1] also names AND / XOR launches and a 50/50 XOR + AND compound mix (a compound launch interleaves the
    # two kinds over the same input pairs, encirc/engine.py:300-320): same launch size, one timed launch each
    by_kind = {}
    if job.rank == 0 and job.world == 1:
        pairs = k // 2
        for name, kind_ids in (("AND", np.full(k, 0, np.uint8)), ("XOR", np.full(k, 4, np.uint8)),
                               ("XOR+AND compound mix", np.tile(np.array([4, 0], np.uint8), pairs))):
            kd = torch.from_numpy(kind_ids).to(dev)
            if name.endswith("mix"):  # jobs 2i and 2i+1 share the input pair i
                xi = torch.arange(pairs, dtype=torch.int32, device=dev).repeat_interleave(2)
                xm, ym = xi.contiguous(), (xi + k).contiguous()
            else:
                xm, ym = xr, yr

            def part(kd=kd, xm=xm, ym=ym):
                ctx.call("tfb_gate_launch", pool.data_ptr(), kd.data_ptr(), xm.data_ptr(), ym.data_ptr(), orow.data_ptr(),
                         len(kd), job.stream)

            part()
            by_kind[name] = len(kd) / (job.timed(part, 1) * 1e-3)

    # dominant kernel alone (K1: fused blind rotation) for the roofline
    ext = torch.empty((k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)

    def k1_only():
        ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kinds.data_ptr(), xr.data_ptr(), yr.data_ptr(),
                 ext.data_ptr(), k, job.stream)

    k1_only()
    k1_reps = max(2, args.steps // 2)
    k1_ms = job.timed(k1_only, k1_reps) / k1_reps
    del ext

    # end to end through the host-buffer entry point (pinned host memory, copies inside the timed region)
    hx = torch.from_numpy(words[0].view(np.int32)).pin_memory()
    hy = torch.from_numpy(words[1].view(np.int32)).pin_memory()
    hk = torch.full((k,), NAND, dtype=torch.uint8).pin_memory()
    hout = torch.empty((k, n + 1), dtype=torch.int32).pin_memory()

    def e2e_step():
        ctx.call("tfb_gate_launch_host", hx.data_ptr(), hy.data_ptr(), hk.data_ptr(), hout.data_ptr(), k)

    e2e_warm, e2e_steps = min(args.warmup, 2), max(2, min(args.steps, 3))
    for _ in range(e2e_warm):
        e2e_step()
    job.fence()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    job.fence()
    e2e_s = job.max_over_ranks(time.perf_counter() - t0)
    out_words = hout.numpy().view(np.uint32)
    e2e_phase = out_words[:, -1] - out_words[:, :-1] @ job.key.bits.astype(np.uint32)
    e2e_ok = job.all_true(np.array_equal(((e2e_phase > 0) & (e2e_phase < 2**31)).astype(int), 1 - (bits[0] & bits[1])))
    del pool
    return {
        "value": value, "ms_per_step": total_ms / args.steps, "scaling": "weak", "clocks": clocks.summary(),
        "gpu_launches": int(gpu_launches), "correct": correct, "k1_ms": k1_ms, "sweep": sweep, "by_kind": by_kind,
        "e2e": {"value": job.world * k * e2e_steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(2 * k * (n + 1) * 4 + k), "d2h_bytes_per_step": int(k * (n + 1) * 4),
                "api": "tfb_gate_launch_host (C ABI, pinned host buffers)", "correct": e2e_ok},
    }


def k1_roofline_probe(job: Job, k: int = 1 << 16) -> float:
    """ms of one K1 launch of 2**16 gates (the dominant kernel of every workload)."""
    torch, ctx, dev, _cabi = job.torch, job.ctx, job.dev, job._cabi
    n = job.key.params.m
    _, words = synth_inputs(job.key.bits, 4096, ENGINE_SEED)
    pool = torch.zeros((2 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
    rep = torch.arange(k, device=dev) % 4096
    pool[:k, : n + 1] = torch.from_numpy(words[0].view(np.int32)).to(dev)[rep]
    pool[k:, : n + 1] = torch.from_numpy(words[1].view(np.int32)).to(dev)[rep]
    kinds = torch.full((k,), NAND, dtype=torch.uint8, device=dev)
    idx = torch.arange(2 * k, dtype=torch.int32, device=dev)
    ext = torch.empty((k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)

    def k1_only():
        ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kinds.data_ptr(), idx[:k].data_ptr(), idx[k:].data_ptr(),
                 ext.data_ptr(), k, job.stream)

    k1_only()
    return job.timed(k1_only, 2) / 2


def sharded_operands(job: Job, workload: str, lanes: int, width: int):
    """Root: random plaintexts, encrypted on the device, packed operand words as device tensors."""
    eng = job.eng
    rng = np.random.default_rng((ENGINE_SEED, 2))
    count = lanes * lanes if workload == "matmul16" else lanes
    plain = [rng.integers(0, 1 << width, size=count, dtype=np.uint64) for _ in range(2)]
    if job.rank != 0:
        return plain, None, None
    packed = []
    for values in plain:
        bits = ((values[:, None] >> np.arange(width, dtype=np.uint64)[None, :]) & 1).astype(np.uint8)
        rows, owner = eng.encrypt_rows(bits.reshape(-1))
        packed.append(eng.export_words_tensor(rows).reshape(count, width, -1).clone())
        del owner
    return plain, packed[0], packed[1]


def sharded_workload(job: Job, workload: str, lanes: int, width: int, steps: int, warmup: int, host_e2e: bool) -> dict:
    """configs[4]: one whole sharded operation per step (strong scaling)."""
    from paper_2005_01945_b200 import sharding

    torch, eng = job.torch, job.eng
    plain, u_t, v_t = sharded_operands(job, workload, lanes, width)
    out_width = 2 * width if workload == "vec_mul" else width

    def op(u, v, as_numpy=False):
        if workload == "vec_add":
            return sharding.sharded_vec_add(eng, u, v, lanes, width, as_numpy=as_numpy, with_stats=True)
        if workload == "vec_mul":
            return sharding.sharded_vec_mul(eng, u, v, lanes, width, as_numpy=as_numpy, with_stats=True)
        return sharding.sharded_mat_mul(eng, u, v, lanes, lanes, lanes, width, as_numpy=as_numpy, with_stats=True)

    state = {}

    def step():
        eng.reset_stats()
        state["out"], state["stats"] = op(u_t, v_t)
        eng.synchronize()

    for _ in range(warmup):
        step()
    launches0 = job.ctx.kernel_launches
    with ClockSampler(job.local) as clocks:
        total_ms = job.timed(step, steps)
    gpu_launches = job.ctx.kernel_launches - launches0
    stats = state["stats"]
    # verification on the root: decrypt the gathered result words
    ok = True
    if job.rank == 0:
        words = state["out"].cpu().numpy().view(np.uint32)
        ph = words[..., -1] - words[..., :-1] @ job.key.bits.astype(np.uint32)
        bits = ((ph > 0) & (ph < 2**31)).astype(np.uint64)
        got = (bits << np.arange(out_width, dtype=np.uint64)[None, :]).sum(axis=1)
        a, b = plain
        if workload == "vec_add":
            want = (a + b) % (1 << width)
        elif workload == "vec_mul":
            want = a * b
        else:
            A, B = a.reshape(lanes, lanes).astype(object), b.reshape(lanes, lanes).astype(object)
            want = np.array([[int(sum(A[i, t] * B[t, j] for t in range(lanes))) % (1 << width) for j in range(lanes)]
                             for i in range(lanes)], dtype=np.uint64).reshape(-1)
        ok = bool(np.array_equal(got, want.astype(np.uint64)))
    ok = job.all_true(ok)
    res = {
        "value": stats.bootstraps * steps / (total_ms * 1e-3), "ms_per_step": total_ms / steps, "scaling": "strong",
        "seconds_per_op": total_ms / steps * 1e-3, "clocks": clocks.summary(), "gpu_launches": int(gpu_launches),
        "correct": ok, "logical_stats": stats.as_record(), "lanes": lanes, "width": width,
        "kernel_launch_levels_last_op": eng.physical_launches,
    }
    if host_e2e:
        # the same operation from HOST operand words (pinned) to HOST result words: H2D of both operands on the
        # root before the scatter and D2H of the gathered result inside the timed region
        hu = hv = None
        if job.rank == 0:
            hu, hv = u_t.cpu().pin_memory(), v_t.cpu().pin_memory()
        job.fence()
        t0 = time.perf_counter()
        out, st = op(hu, hv, as_numpy=True)
        job.fence()
        dt = job.max_over_ranks(time.perf_counter() - t0)
        nbytes = int(u_t.numel() * 4) if job.rank == 0 else 0
        res["e2e"] = {"value": st.bootstraps / dt, "unit": UNIT, "h2d_bytes_per_step": 2 * nbytes,
                      "d2h_bytes_per_step": int(out.nbytes) if out is not None else 0,
                      "api": f"sharding.sharded_{'mat_mul' if workload == 'matmul16' else workload} (host words in, host words out)",
                      "seconds_per_op": dt}
    return res


def time_circuits(job: Job) -> dict:
    """The second half of BASELINE.json's metric: 16/32-bit encrypted add / multiply through the public engine API,
    results verified; latency of ONE operation (depth-bound: 3n / 1 + 6n*ceil(log2 n) logical launches, run as
    2n+1 / ~138 dependent kernel-launch levels) and throughput of a batch of independent operations (vec_add /
    vec_mul lanes), each beside the reference's CPU engine timed in this run."""
    from paper_2005_01945_b200 import (
        add_bitwise, decrypt_int, decrypt_vector, encrypt_int, encrypt_vector, mul_karatsuba, mul_naive, vec_add, vec_mul,
    )

    eng = job.eng
    rng = np.random.default_rng((ENGINE_SEED, 2))
    out = {}
    for n in (16, 32):
        a, b = (int(v) for v in rng.integers(0, 1 << n, size=2, dtype=np.uint64))
        x, y = encrypt_int(eng, a, n), encrypt_int(eng, b, n)
        for name, fn, want in ((f"add{n}", add_bitwise, (a + b) % (1 << n)), (f"mul{n}", mul_naive, a * b),
                               (f"karatsuba{n}", mul_karatsuba, a * b)):
            fn(encrypt_int(eng, 3, n), encrypt_int(eng, 5, n))  # warm the launch path (first use of each kernel variant)
            eng.synchronize()
            best = None
            for _ in range(3):
                eng.reset_stats()
                eng.physical_launches = 0
                t0 = time.perf_counter()
                res = fn(x, y)
                eng.synchronize()
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            out[name] = {"seconds": best, "ops_per_s": 1.0 / best, "bootstraps": eng.stats.bootstraps,
                         "launches": eng.stats.batch_launches, "kernel_launch_levels": eng.physical_launches,
                         "correct": decrypt_int(eng, res) == want}
    for name, lanes, fn in (("add32_x256", 256, vec_add), ("mul32_x16", 16, vec_mul)):
        u = [int(v) for v in rng.integers(0, 1 << 32, size=lanes, dtype=np.uint64)]
        v = [int(v) for v in rng.integers(0, 1 << 32, size=lanes, dtype=np.uint64)]
        U, V = encrypt_vector(eng, u, 32), encrypt_vector(eng, v, 32)
        eng.synchronize()
        eng.reset_stats()
        t0 = time.perf_counter()
        res = fn(U, V)
        eng.synchronize()
        dt = time.perf_counter() - t0
        want = [(p + q) % (1 << 32) for p, q in zip(u, v)] if fn is vec_add else [p * q for p, q in zip(u, v)]
        out[name] = {"seconds": dt, "ops_per_s": lanes / dt, "bootstraps": eng.stats.bootstraps,
                     "correct": decrypt_vector(eng, res) == want}
    cpu = reference_circuit_seconds()
    if cpu is None:
        out["reference_cpu"] = {"unavailable": "oracle/_ref not staged"}
    else:
        out["reference_cpu"] = cpu
        ratios = {}
        for name in ("add16", "mul16", "karatsuba16", "add32", "mul32", "karatsuba32", "add32_x256", "mul32_x16"):
            best_cpu = min(cpu[w][name]["seconds"] for w in cpu if w.startswith("workers_"))
            ratios[name] = best_cpu / out[name]["seconds"]
        out["speedup_vs_reference_cpu"] = ratios  # > 1: the GPU finishes sooner than the reference's CPU oracle engine
    out["paper_gtx1080_seconds"] = {"add32": 1.99, "mul32": 33.99, "source": "BASELINE.md section 2 (PAPER.md:802-810, 862-864)"}
    return out


def time_latency(job: Job, calls: int = 1000) -> dict:
    """configs[0]: one bootstrapped NAND / AND / XOR gate, submit -> result resident, median over `calls`
    sequential eval_gate calls through the engine API."""
    from paper_2005_01945_b200 import GateKind

    eng = job.eng
    x, y = eng.encrypt(1), eng.encrypt(0)
    eng.synchronize()
    out = {}
    for kind in (GateKind.NAND, GateKind.AND, GateKind.XOR):
        for _ in range(10):
            eng.eval_gate(kind, x, y)
            eng.synchronize()
        ts = []
        for _ in range(calls):
            t0 = time.perf_counter()
            bit = eng.eval_gate(kind, x, y)
            eng.synchronize()
            ts.append(time.perf_counter() - t0)
        out[kind.value] = {"median_ms": float(np.median(ts)) * 1e3, "p90_ms": float(np.percentile(ts, 90)) * 1e3,
                           "calls": calls, "correct": eng.decrypt(bit) == {"NAND": 1, "AND": 0, "XOR": 1}[kind.value]}
    return out


def run_b200(args) -> None:
    job = Job(args)
    _cabi = job._cabi
    n = job.key.params.m
    if args.workload == "gates":
        head = gates_workload(job)
        k1_ms = head.pop("k1_ms")
    else:
        lanes, width = sharded_shape(args)
        head = sharded_workload(job, args.workload, lanes, width, args.steps, args.warmup, host_e2e=True)
        k1_ms = k1_roofline_probe(job)
    sharded = None
    if args.workload == "gates" and not args.no_sharded:
        # one strong-scaling figure on every default line: vec_add 4096 x 32-bit (655,360 bootstraps)
        sharded = {"vec_add": sharded_workload(job, "vec_add", args.lanes or 4096, 32, 1, 1, host_e2e=False)}
    if job.rank != 0:
        job.close()
        return

    peaks = _cabi.measure_peaks(job.local)
    k1_gates = 1 << 16 if args.workload != "gates" else args.batch
    k1_tflops = k1_gates * FLOP_PER_GATE / (k1_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "k1_dram_bytes_per_launch.json")
    if os.path.exists(prof):
        with open(prof) as f:
            rec = json.load(f)
        traffic = rec.get("dram_bytes_per_launch")
        traffic_src = (f"stored ncu --set full capture of this kernel at {rec.get('gates_per_launch')} gates per launch "
                       f"(dram__bytes_read.sum + dram__bytes_write.sum), {rec.get('source', 'profiles/')}; "
                       "not re-measured in this run")
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": job.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": head["scaling"], "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": config(args, job.world), "clocks": head["clocks"], "e2e": head["e2e"],
        "gpu_launches": head["gpu_launches"], "correct": head["correct"],
        "roofline": {
            "kernel": "k_gate_bootstrap_warp (K1d: fused linear form + blind rotation + sample extract, one gate per warp)",
            "bound": "fp64", "achieved": k1_tflops, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
            "frac": k1_tflops / peaks["fp64_tflops"], "traffic": traffic, "traffic_source": traffic_src,
            "flop_per_gate": FLOP_PER_GATE, "ms_per_launch": k1_ms, "gates_per_launch": k1_gates,
            # the same launch rated by the work a plain (not unrolled) CMux loop would need: what rounds 1-2a reported
            "flop_per_gate_plain_cmux": FLOP_PER_GATE_PLAIN_CMUX,
            "frac_at_plain_cmux_count": k1_gates * FLOP_PER_GATE_PLAIN_CMUX / (k1_ms * 1e-3) / 1e12 / peaks["fp64_tflops"],
            "share_of_step": (k1_ms / head["ms_per_step"]) if args.workload == "gates" else None,
            "peak_source": "measured in this run: dependent-free DFMA loop on all SMs (tfb_measure_peaks); "
                           "MEASURED_PEAKS.json has no FP64 figure",
            "hbm_algorithmic_bytes_per_gate": 3 * (n + 1) * 4 + 2 * 1025 * 4, "hbm_peak_gbs": _measured_hbm(),
        },
    }
    for extra in ("logical_stats", "seconds_per_op", "lanes", "width", "kernel_launch_levels_last_op"):
        if extra in head:
            line[extra] = head[extra]
    if head.get("sweep"):
        line["sweep"] = {"unit": UNIT, "gates_per_s_by_launch_size": head["sweep"],
                         "gates_per_s_by_kind_at_full_launch": head.get("by_kind", {})}
    if sharded is not None:
        line["sharded"] = sharded
    if job.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = reference_gate_rates(1 << 14, 2, 1)
        real_value, threads, real_ok = time_real_bootstrap_cpu(256)
        line["cpu_real_bootstrap"] = {
            "value": real_value, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "256 NAND gates, oracle/tfhe_gate_oracle.c double-FFT path (real TFHE bootstrap + key switch); "
                      "NOT the reference -- the like-for-like CPU comparator", "correct": real_ok}
    if job.world == 1 and not args.no_circuits:
        line["circuits"] = time_circuits(job)
        line["latency"] = time_latency(job)
    print(json.dumps(line))
    job.close()


def _measured_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f)["hbm_gbs"]
    except Exception:
        return 6650.0  # fallback stated in B200_PROFILING.md


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "RANK" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start one rank per GPU ourselves
        import socket

        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    run_b200(args)


if __name__ == "__main__":
    main()
