mkdir -p gpurun_out/s8
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s8/smoke.log 2>&1; tail -2 gpurun_out/s8/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/s8/bench.json 2> gpurun_out/s8/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s8/bench_ref.json 2> gpurun_out/s8/bench_ref.err
timeout 300 python tools/k1c_latency.py > gpurun_out/s8/latency.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/s8/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/s8/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap_warp -s 1 -c 1 -f -o gpurun_out/s8/k1d python tests/gpu_profile_target.py --k 65536 --reps 2 > gpurun_out/s8/ncu_k1d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap_pair -s 1 -c 1 -f -o gpurun_out/s8/k1e python tests/gpu_profile_target.py --k 64 --reps 2 > gpurun_out/s8/ncu_k1e.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap_warp_mid -s 1 -c 1 -f -o gpurun_out/s8/k1d_mid python tests/gpu_profile_target.py --k 592 --reps 2 > gpurun_out/s8/ncu_k1d_mid.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_key_switch_narrow -s 1 -c 1 -f -o gpurun_out/s8/k2n python tests/gpu_profile_target.py --k 2 --reps 2 > gpurun_out/s8/ncu_k2n.log 2>&1
REF_ACCEPT_FULL=1 timeout 1500 python -m pytest tests/test_reference_suite.py -m gpu -x -q > gpurun_out/s8/ref_suite_full.log 2>&1; tail -3 gpurun_out/s8/ref_suite_full.log
python - <<'PY'
import json
d=json.load(open('gpurun_out/s8/bench.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])
print({k:(v.get('seconds') if isinstance(v,dict) else v) for k,v in d['circuits'].items() if k!='reference_cpu'})
PY
cat gpurun_out/s8/latency.log
