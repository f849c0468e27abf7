#!/bin/bash
# GEMM CTA-0 timeline (slots: 0 producer stage issue, 1 MMA stage full, 2 MMA
# stage committed, 7 MMA j-group start, 6 epilogue j-group rowsums ready,
# 3 acc_full seen, 4 acc released, 5 j-group math done).  Needs
# scratch/ab_trace (tools/ab_build.py with -DLANCE_PROFILING -DLANCE_GEMM_TRACE).
set -u
TAG=${1:-trace}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for L in "512 7 256" "256 14 256" "64 56 256"; do
  set -- $L
  LANCE_LIB_PATH=scratch/ab_trace/liblance_b200.so LANCE_GEMM_TRACE=$OUT/tr timeout 120 python scratch/trace_run.py $1 $2 $3 >> $OUT/log.txt 2>&1
done
ls -la $OUT
