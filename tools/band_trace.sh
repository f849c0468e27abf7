#!/bin/bash
# Trace-enabled build of the band kernels, one R64 layer, dump the trace via a ctypes hook.
set -u
TAG=$1
OUT=gpurun_out/$TAG
mkdir -p $OUT
D=/tmp/bt; mkdir -p $D
for f in lance_input lance_band lance_filter lance_gemm lance_abi; do
  nvcc -DLANCE_BAND_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -c paper_2003_08646_b200/csrc/$f.cu -o $D/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/liblance_b200.so $D/*.o
LANCE_LIB_PATH=$D/liblance_b200.so timeout 120 python scratch/band_trace_run.py 64 56 256 $OUT/trace_c64.bin > $OUT/log.txt 2>&1
LANCE_LIB_PATH=$D/liblance_b200.so timeout 120 python scratch/band_trace_run.py 512 7 256 $OUT/trace_c512.bin >> $OUT/log.txt 2>&1
echo done
