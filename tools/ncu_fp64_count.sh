#!/bin/bash
# FP64-pipe warp instructions and duration of one K1d wave (1776 gates), per library given on the command line
for lib in "$@"; do
  echo "== $lib"
  ncu --metrics smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:k_gate_bootstrap_warp -c 1 python tools/k1_ab.py --k 1776 --kernels 4 --reps 1 --lib $lib 2>&1 | grep -E "smsp__|gpu__time|sm__pipe|l1tex" 
done
