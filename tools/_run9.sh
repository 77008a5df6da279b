echo "== 6 slots"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 2>&1 | tail -1
echo "== 5 slots"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 --lib tools/lib_slots5.so 2>&1 | tail -1
timeout 300 python tools/k1d_warp_sweep.py 2>&1 | grep -E "k1d_w(4|8|12) |k1d_w[1-3] "
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
