mkdir -p gpurun_out/s6
echo "== base"; timeout 300 python tools/k1c_latency.py 2>&1 | grep -E "k=   1 |k=  64|k=  74"
echo "== prefetch"; timeout 300 python tools/k1c_latency.py tools/lib_k1e_pf1.so 2>&1 | grep -E "K1e.*(k=   1 |k=  64)"
timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 2>&1 | tail -1
