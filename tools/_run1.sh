set -x
mkdir -p gpurun_out/s3
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/s3/pytest.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s3/bench_ref.json 2> gpurun_out/s3/bench_ref.err
timeout 300 python tools/k1c_latency.py > gpurun_out/s3/latency.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s3/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/s3/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap_warp -s 1 -c 1 -f -o gpurun_out/s3/k1d python tests/gpu_profile_target.py --k 14208 --reps 2 > gpurun_out/s3/ncu_k1d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap_pair -s 1 -c 1 -f -o gpurun_out/s3/k1e python tests/gpu_profile_target.py --k 64 --reps 2 > gpurun_out/s3/ncu_k1e.log 2>&1
tail -3 gpurun_out/s3/pytest.log; cat gpurun_out/s3/bench.json | head -c 3000; cat gpurun_out/s3/latency.log
