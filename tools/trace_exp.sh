#!/bin/bash
# GEMM timeline of the R64 layer with the epilogue on (exp 0) and skipped (exp 1).
set -u
OUT=gpurun_out/${1:-trexp}
mkdir -p $OUT
for e in 0 1 16 18; do
  LANCE_GEMM_EXP=$e LANCE_LIB_PATH=scratch/ab_trace/liblance_b200.so LANCE_GEMM_TRACE=$OUT/e$e timeout 120 python scratch/trace_run.py 64 56 256 >> $OUT/log.txt 2>&1
done
ls $OUT
