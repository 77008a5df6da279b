mkdir -p gpurun_out/s9
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_bootstrap_warp -c 1 -f -o gpurun_out/s9/k1d python tests/gpu_profile_target.py --k 63936 --reps 1 > gpurun_out/s9/ncu_k1d.log 2>&1
tail -2 gpurun_out/s9/ncu_k1d.log
