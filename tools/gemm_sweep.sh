#!/bin/bash
# GEMM stage-shape sweep (profiling build knobs): LANCE_GEMM_STAGE x LANCE_GEMM_UNITS,
# all four ResNet-18 shapes at batch 256.
set -u
OUT=gpurun_out/${1:-gsweep}
mkdir -p $OUT
LIB=scratch/ab_prof/liblance_b200.so
for st in 1 0; do for un in 1 2 4; do
  LANCE_LIB_PATH=$LIB LANCE_GEMM_STAGE=$st LANCE_GEMM_UNITS=$un timeout 300 python bench.py --layers 0,4,7,10 --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/s${st}_u${un}.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/s${st}_u${un}.json')); pl=d['roofline']['per_layer']
print('stage=$st units=$un', [l['us_per_forward'][2] for l in pl])"
done; done
