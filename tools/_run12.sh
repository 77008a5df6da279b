for v in stag1000 stag3000 stag6000; do echo "== $v"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 --lib tools/lib_$v.so 2>&1 | tail -1; done
echo "== base"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 2>&1 | tail -1
