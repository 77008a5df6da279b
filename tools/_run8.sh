echo "== K1e nocombine"; timeout 300 python tools/k1c_latency.py tools/lib_nocombine.so 2>&1 | grep -E "K1e.*(k=   1 |k=  64)"
for v in relaxed slots4; do echo "== K1d $v"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 --lib tools/lib_$v.so 2>&1 | tail -1; done
echo "== K1d base"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 2>&1 | tail -1
