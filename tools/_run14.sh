for v in base noearly nopretest neither; do
  lib=""; [ $v != base ] && lib="--lib tools/lib_$v.so"
  echo "== $v"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208,592 --reps 3 $lib 2>&1 | grep "^4 "
done
