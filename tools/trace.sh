#!/bin/bash
set -u
TAG=${1:-trace}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for e in 0 3; do
  LANCE_GEMM_EXP=$e LANCE_GEMM_TRACE=$OUT/tr_e$e timeout 120 python scratch/trace_run.py 64 56 256 >> $OUT/log.txt 2>&1
  LANCE_GEMM_EXP=$e LANCE_GEMM_TRACE=$OUT/tr_e$e timeout 120 python scratch/trace_run.py 512 7 256 >> $OUT/log.txt 2>&1
done
echo done
