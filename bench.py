"""bench.py -- bootstrapped gates/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--batch 65536]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N ... bench.py --gpus N ...

A "step" is one launch of `batch` independent bootstrapped NAND gates at the
reference's default parameter set (BASELINE.json configs[1]: 2**16 ciphertexts
per launch), synthetic random plaintexts, inputs resident in HBM.  `value` is
whole-job gates/s over N GPUs (weak scaling: every rank runs its own 2**16-gate
launch per step; gates are independent, so there is no data-path collective --
NCCL only broadcasts the evaluation keys and reduces the timing / checks).
`e2e` is the same metric through the C ABI's host-buffer entry point with the
host<->device copies inside the timed region.  `roofline` is the fused
bootstrap kernel against the FP64 pipe (this path is bound by the
FP64 transform+MAC work, not HBM and not tensor cores), with the DFMA peak
measured in the same run.  `cpu_baseline` times the reference's own CPU path
(oracle/encirc_port.py, pinned bit-exactly to the reference) on a bounded
sample; `cpu_real_bootstrap` times our C restatement of the REAL bootstrap, the
like-for-like CPU comparator (the reference's "bootstrap" is a decrypt /
re-encrypt oracle, not TFHE).
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
# 500 iterations x (6 negacyclic transforms of 26,112 FLOP + 8 x 512 complex MACs) per gate
FLOP_PER_GATE = 500 * (6 * 26112 + 32768)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=1 << 16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-circuits", action="store_true")
    return ap.parse_args()


def config(args, n_gpus):
    return {
        "workload": "BASELINE configs[1]: batched independent NAND gates, one launch per step",
        "batch_per_gpu": args.batch,
        "params": "m=500 alpha=2^-15 w=32 mu=1/8; ring N=1024 k=1 l=2 Bg=2^10 ks t=8 base=4",
        "parallelism": f"gates sharded over {n_gpus} GPU(s), no data-path collective",
        "l2": "inputs (2 x batch x 2 KiB = 268 MB) exceed the 126 MB L2; no flush needed",
    }


def synth_inputs(key_bits: np.ndarray, k: int, seed: int):
    """Vectorised fresh encryptions of uniform random bits (same distribution
    as encirc/torus.py:254-271; the draw order differs, which only matters to
    the parity tests, not to throughput)."""
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
# reference arm / CPU baselines
# ------------------------------------------------------------------------------------------

def time_reference_cpu(k: int, steps: int, warmup: int):
    """The reference's own CPU path (oracle-LWE engine port) on `k` NAND gates
    per step in one launch (max_batch = k), encryption outside the timed region
    like encirc/bench.py:179-190."""
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
    got = np.array([eng.decrypt(c) for c in outs[:4096]])
    ok = bool(np.array_equal(got, 1 - (bits[0, :4096] & bits[1, :4096])))
    return k * steps / dt, dt / steps, ok


def time_real_bootstrap_cpu(sample: int):
    """Our C restatement of the real TFHE bootstrap (double-precision FFT path),
    all host threads: the like-for-like CPU comparator."""
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


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    k = min(args.batch, 1 << 16)
    value, per_step, ok = time_reference_cpu(k, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{k} NAND gates per step in one launch; oracle/encirc_port.py (the reference's "
                                   "decrypt/re-encrypt oracle engine, single-threaded numpy: its thread pool gives no "
                                   "speed-up under the GIL, SURVEY 2.3)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "correct": ok,
        "note": "the reference CPU path is a key-holding oracle (one 500-long dot product + RNG per gate), not a TFHE bootstrap",
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------

def run_b200(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2005_01945_b200 import LweParams, _cabi, generate_evaluation_keys, keygen
    from paper_2005_01945_b200.keys import RingParams

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    distributed = "RANK" in os.environ and "WORLD_SIZE" in os.environ  # launched by torch.distributed.run
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    key = keygen(LweParams(), seed=KEY_SEED)
    n, k = key.params.m, args.batch
    ring = RingParams()
    ctx = _cabi.Context(local, n, key.params.mu.word, ring)
    stream = torch.cuda.current_stream(dev).cuda_stream
    # evaluation keys: generated on rank 0, broadcast raw over NCCL, transformed on every GPU (kernel K3)
    if distributed:
        bk_t = torch.empty((n, ring.rows, 2, ring.N), dtype=torch.int32, device=dev)
        ksk_t = torch.empty((ring.N, ring.ks_t, n + 1), dtype=torch.int32, device=dev)
        if rank == 0:
            ek = generate_evaluation_keys(key, seed=ENGINE_SEED, ring=ring)
            bk_t.copy_(torch.from_numpy(ek.bk))
            ksk_t.copy_(torch.from_numpy(ek.ksk))
        dist.broadcast(bk_t, 0)
        dist.broadcast(ksk_t, 0)
        ctx.call("tfb_load_keys", bk_t.data_ptr(), ksk_t.data_ptr(), 1, stream)
        del bk_t, ksk_t
    else:
        ek = generate_evaluation_keys(key, seed=ENGINE_SEED, ring=ring)
        ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, stream)

    bits, words = synth_inputs(key.bits, k, ENGINE_SEED + rank)
    pool = torch.zeros((3 * k, _cabi.ROW_STRIDE), dtype=torch.int32, device=dev)
    pool[:k, : n + 1] = torch.from_numpy(words[0].view(np.int32)).to(dev)
    pool[k : 2 * k, : n + 1] = torch.from_numpy(words[1].view(np.int32)).to(dev)
    kinds = torch.full((k,), NAND, dtype=torch.uint8, device=dev)
    idx = torch.arange(3 * k, dtype=torch.int32, device=dev)
    xr, yr, orow = idx[:k], idx[k : 2 * k], idx[2 * k :]
    key_bits_t = torch.from_numpy(key.bits.astype(np.uint32).view(np.int32)).to(dev)

    def step():
        ctx.call("tfb_gate_launch", pool.data_ptr(), kinds.data_ptr(), xr.data_ptr(), yr.data_ptr(), orow.data_ptr(),
                 k, stream)

    def fence():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fence()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        fence()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    for _ in range(args.warmup):
        step()
    launches0 = ctx.kernel_launches
    with ClockSampler(local) as clocks:
        total_ms = timed(step, args.steps)
    gpu_launches = ctx.kernel_launches - launches0
    value = world * k * args.steps / (total_ms * 1e-3)

    # correctness of the timed work: every output of the last step decrypts to NAND
    ph = torch.empty(k, dtype=torch.int32, device=dev)
    ctx.call("tfb_rows_phase", pool.data_ptr(), orow.data_ptr(), key_bits_t.data_ptr(), ph.data_ptr(), k, stream)
    phase = ph.cpu().numpy().view(np.uint32)
    correct = bool(np.array_equal(((phase > 0) & (phase < 2**31)).astype(int), 1 - (bits[0] & bits[1])))
    if distributed:
        flag = torch.tensor([int(correct)], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        correct = bool(flag.item())

    # dominant kernel alone (K1: fused blind rotation) for the roofline
    ext = torch.empty((k, _cabi.EXT_STRIDE), dtype=torch.int32, device=dev)

    def k1_only():
        ctx.call("tfb_debug_blind_rotate", pool.data_ptr(), kinds.data_ptr(), xr.data_ptr(), yr.data_ptr(),
                 ext.data_ptr(), k, stream)

    k1_only()
    k1_reps = max(2, args.steps // 2)
    k1_ms = timed(k1_only, k1_reps) / k1_reps
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
    fence()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    fence()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = world * k * e2e_steps / float(e2e_s.item())
    out_words = hout.numpy().view(np.uint32)
    e2e_phase = out_words[:, -1] - out_words[:, :-1] @ key.bits.astype(np.uint32)
    e2e_ok = bool(np.array_equal(((e2e_phase > 0) & (e2e_phase < 2**31)).astype(int), 1 - (bits[0] & bits[1])))

    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return

    peaks = _cabi.measure_peaks(local)
    k1_tflops = k * FLOP_PER_GATE / (k1_ms * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k1_dram_bytes_per_launch.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+u32", "data": "synthetic", "config": config(args, world),
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(2 * k * (n + 1) * 4 + k),
                "d2h_bytes_per_step": int(k * (n + 1) * 4), "api": "tfb_gate_launch_host (C ABI, pinned host buffers)",
                "correct": e2e_ok},
        "gpu_launches": int(gpu_launches),
        "correct": correct,
        "roofline": {
            "kernel": "k_gate_bootstrap_warp (K1d: fused linear form + blind rotation + sample extract, one gate per warp)",
            "bound": "fp64", "achieved": k1_tflops, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
            "frac": k1_tflops / peaks["fp64_tflops"], "traffic": traffic,
            "flop_per_gate": FLOP_PER_GATE, "ms_per_launch": k1_ms, "share_of_step": k1_ms / (total_ms / args.steps),
            "peak_source": "measured in this run: dependent-free DFMA loop on all SMs (tfb_measure_peaks); "
                           "MEASURED_PEAKS.json has no FP64 figure",
            "hbm": {"algorithmic_bytes_per_gate": 3 * (n + 1) * 4 + 2 * 1025 * 4,
                    "achieved_gbs": k * (3 * (n + 1) * 4 + 2 * 1025 * 4) / (total_ms / args.steps * 1e-3) / 1e9,
                    "peak_gbs": _measured_hbm()},
        },
    }
    if world == 1 and not args.no_cpu_baseline:
        ref_k = 1 << 14
        cpu_value, _, cpu_ok = time_reference_cpu(ref_k, 2, 1)
        line["cpu_baseline"] = {
            "value": cpu_value, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{ref_k} NAND gates per launch, 2 timed launches, oracle/encirc_port.py "
                      "(reference decrypt/re-encrypt oracle engine; single-threaded numpy)", "correct": cpu_ok}
        real_value, threads, real_ok = time_real_bootstrap_cpu(256)
        line["cpu_real_bootstrap"] = {
            "value": real_value, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "256 NAND gates, oracle/tfhe_gate_oracle.c double-FFT path (real TFHE bootstrap + key switch); "
                      "NOT the reference -- the like-for-like CPU comparator", "correct": real_ok}
    if world == 1 and not args.no_circuits:
        line["circuits"] = time_circuits(local)
    print(json.dumps(line))
    if distributed:
        dist.destroy_process_group()


def time_circuits(device: int) -> dict:
    """The second half of BASELINE.json's metric: 32-bit encrypted add / multiply through the
    public engine API, results verified.  Latency-bound: 96 and 961 launches as the reference counts them,
    which the engine's levelised execution runs as 65 and 138 dependent kernel-launch levels."""
    from paper_2005_01945_b200 import (
        B200Engine, LweParams, PoolConfig, WorkerPool, add_bitwise, decrypt_int, encrypt_int, keygen, mul_naive,
    )

    eng = B200Engine(keygen(LweParams(), seed=KEY_SEED), seed=ENGINE_SEED, device=device,
                     pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)))
    rng = np.random.default_rng((ENGINE_SEED, 2))
    a, b = (int(v) for v in rng.integers(0, 1 << 32, size=2, dtype=np.uint64))
    x, y = encrypt_int(eng, a, 32), encrypt_int(eng, b, 32)
    out = {}
    for name, fn, want in (("add32", add_bitwise, (a + b) % (1 << 32)), ("mul32", mul_naive, a * b)):
        fn(encrypt_int(eng, 3, 32), encrypt_int(eng, 5, 32))  # warm the launch path (first use of each kernel variant)
        eng.synchronize()
        eng.reset_stats()
        eng.physical_launches = 0
        t0 = time.perf_counter()
        res = fn(x, y)
        eng.synchronize()
        dt = time.perf_counter() - t0
        out[name] = {"seconds": dt, "ops_per_s": 1.0 / dt, "bootstraps": eng.stats.bootstraps,
                     "launches": eng.stats.batch_launches, "kernel_launch_levels": eng.physical_launches,
                     "correct": decrypt_int(eng, res) == want}
    out["reference_cpu_seconds"] = {"add32": 0.018, "mul32": 0.281,
                                    "source": "BASELINE.md section 3: the reference's oracle engine on the build "
                                              "container (not a bootstrap)"}
    out["paper_gtx1080_seconds"] = {"add32": 1.99, "mul32": 33.99, "source": "BASELINE.md section 2 (PAPER.md:802-810, 862-864)"}
    return out


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
