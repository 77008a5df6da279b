#!/bin/bash
# The measurement pass behind profiles/README.md, for one B200 (run from the repo root, e.g. under gpurun):
#   bash tools/gpu_measure.sh [outdir]
# GPU tests, smoke, both bench arms, K1 latency, launch list, `ncu --set full` of every hot kernel, compute-sanitizer
# on the smallest launches, and the condensed summaries tools/ncu_summary.py writes.  Nothing here is a bench value
# if it ran under a profiler: bench.json / bench_ref.json are the unprofiled runs.
out=${1:-gpurun_out/measure}; mkdir -p "$out"
(time timeout 1500 python -m pytest tests -m gpu -x -q) > "$out/pytest.log" 2>&1; tail -3 "$out/pytest.log"
python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; tail -1 "$out/smoke.log"
timeout 600 python bench.py --steps 3 --warmup 3 > "$out/bench.json" 2> "$out/bench.err"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$out/bench_ref.json" 2> "$out/bench_ref.err"
timeout 300 python tools/k1c_latency.py > "$out/latency.log" 2>&1
timeout 300 python tools/k1d_warp_sweep.py > "$out/k1d_warp_sweep.log" 2>&1
timeout 300 python tools/k2_ab.py > "$out/k2_ab.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file "$out/launches.csv" \
    python bench.py --steps 2 --warmup 1 > "$out/bench_under_ncu.log" 2>&1
cap() {  # name, kernel regex, gates
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -c 1 -f -o "$out/$1" \
      python tests/gpu_profile_target.py --k "$3" --reps 1 > "$out/ncu_$1.log" 2>&1
  python tools/ncu_summary.py "$out/$1.ncu-rep" --out "$out/$1_ncu.txt" > /dev/null
}
cap k1d 'k_gate_bootstrap_warp$' 63936   # 36 full waves of twelve gates per SM: one launch
cap k1d_mid k_gate_bootstrap_warp_mid 592
cap k1e k_gate_bootstrap_pair 64
cap k2n k_key_switch_narrow 2
cap k2t k_key_switch_mma 63936
