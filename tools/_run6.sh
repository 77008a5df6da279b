mkdir -p gpurun_out/s7
# race / memory checks on the smallest launches of both K1 kernels and the narrow key switch
cat > /tmp/san.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2005_01945_b200 import _cabi
from paper_2005_01945_b200.keys import generate_evaluation_keys
from paper_2005_01945_b200.torus import LweParams, encrypt_bit, keygen
p = LweParams(m=int(os.environ.get("SAN_N", "20"))); key = keygen(p, seed=11); ek = generate_evaluation_keys(key, seed=11); n = p.m
rng = np.random.default_rng((11, 0))
pack = lambda s: np.concatenate([s.a, [s.b]]).astype(np.uint32)
k = int(os.environ.get("SAN_K", "2"))
xs = np.stack([pack(encrypt_bit(key, g & 1, rng)) for g in range(k)]); ys = np.stack([pack(encrypt_bit(key, (g >> 1) & 1, rng)) for g in range(k)])
ctx = _cabi.Context(0, n, p.mu.word, ek.ring)
ctx.call("tfb_load_keys", ek.bk.ctypes.data, ek.ksk.ctypes.data, 0, None)
kinds = np.full(k, 2, dtype=np.uint8); out = np.zeros((k, n + 1), dtype=np.uint32)
ctx.call("tfb_gate_launch_host", xs.ctypes.data, ys.ctypes.data, kinds.ctypes.data, out.ctypes.data, k)
print("ok", k, n)
PY
for tool in memcheck racecheck; do
  for cfg in "5 2" "4 13"; do set -- $cfg
    echo "== $tool kernel $1 k=$2"; TFB_FORCE_KERNEL=$1 SAN_K=$2 SAN_N=20 timeout 900 compute-sanitizer --tool $tool python /tmp/san.py 2>&1 | tail -4
  done
done > gpurun_out/s7/sanitizer.log 2>&1
cat gpurun_out/s7/sanitizer.log
timeout 900 python tools/noise_stats.py --gates 16777216 --out gpurun_out/s7/noise_64M.json > gpurun_out/s7/noise.log 2>&1; tail -4 gpurun_out/s7/noise.log
timeout 900 python bench.py --workload vec_mul --steps 1 --warmup 0 --no-cpu-baseline --no-circuits > gpurun_out/s7/bench_vec_mul.json 2> gpurun_out/s7/bench_vec_mul.err; head -c 1500 gpurun_out/s7/bench_vec_mul.json; echo
timeout 900 python bench.py --workload matmul16 --steps 1 --warmup 0 --no-cpu-baseline --no-circuits > gpurun_out/s7/bench_matmul16.json 2> gpurun_out/s7/bench_matmul16.err; head -c 1500 gpurun_out/s7/bench_matmul16.json; echo
timeout 900 python bench.py --workload vec_add --steps 2 --warmup 1 --no-cpu-baseline --no-circuits > gpurun_out/s7/bench_vec_add.json 2> gpurun_out/s7/bench_vec_add.err; head -c 1500 gpurun_out/s7/bench_vec_add.json; echo
