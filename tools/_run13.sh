TFB_K1D_W=4 timeout 300 python tools/k1_ab.py --kernels 4 --k 592 --reps 1 --lib tools/lib_phases.so 2>&1 | grep -E "warp|592" | head -8
echo; TFB_K1D_W=8 timeout 300 python tools/k1_ab.py --kernels 4 --k 1184 --reps 1 --lib tools/lib_phases.so 2>&1 | grep -E "warp|1184" | head -5
