#!/bin/bash
# Build scratch/ab_old (an older csrc snapshot) into scratch/ab_old/liblance_b200.so.
set -e
D=scratch/ab_old
for f in lance_input lance_filter lance_gemm lance_abi; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -c $D/$f.cu -o $D/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/liblance_b200.so $D/*.o
