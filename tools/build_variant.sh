#!/bin/bash
# tools/build_variant.sh OUT.so [-DFLAG=..]...   -- A/B builds of libtfhe_b200 for tools/k1_ab.py --lib
out=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -shared -Xcompiler -fPIC "$@" -o "$out" /root/repo/paper_2005_01945_b200/csrc/tfhe_b200.cu
