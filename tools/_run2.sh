mkdir -p gpurun_out/s4
for v in halfkeys nokeys turns; do
  echo "== $v"; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 --lib tools/lib_$v.so 2>&1 | tail -2
done > gpurun_out/s4/k1d_variants.log 2>&1
echo "== base" >> gpurun_out/s4/k1d_variants.log; timeout 300 python tools/k1_ab.py --kernels 4 --k 14208 --reps 3 2>&1 | tail -2 >> gpurun_out/s4/k1d_variants.log
timeout 300 python tools/k1_ab.py --kernels 4 --k 1776 --reps 1 --lib tools/lib_phases.so > gpurun_out/s4/k1d_phases.log 2>&1
timeout 300 python tools/k1_ab.py --kernels 5 --k 64 --reps 1 --lib tools/lib_k1eprobe.so > gpurun_out/s4/k1e_probe.log 2>&1
timeout 600 python tools/noise_stats.py > gpurun_out/s4/noise.log 2>&1
cat gpurun_out/s4/k1d_variants.log; tail -8 gpurun_out/s4/k1d_phases.log; tail -8 gpurun_out/s4/k1e_probe.log; tail -5 gpurun_out/s4/noise.log
