#!/bin/bash
set -u
OUT=gpurun_out/${1:-trjs}
mkdir -p $OUT
for js in 1 0; do
  LANCE_GEMM_JSPLIT=$js LANCE_LIB_PATH=scratch/ab_trace/liblance_b200.so LANCE_GEMM_TRACE=$OUT/js$js timeout 120 python scratch/trace_run.py 512 7 32 >> $OUT/log.txt 2>&1
done
ls $OUT
