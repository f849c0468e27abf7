#!/bin/bash
# Small-M GEMM knobs at the strong-scaling per-rank batches (layers R128/R256/R512).
set -u
OUT=gpurun_out/${1:-gsmall}
mkdir -p $OUT
LIB=scratch/ab_prof/liblance_b200.so
for b in 32 64; do for bn in 64 32 16; do for un in 1 2 4; do for st in 1 0; do
  LANCE_LIB_PATH=$LIB LANCE_GEMM_BN=$bn LANCE_GEMM_UNITS=$un LANCE_GEMM_STAGE=$st timeout 300 python bench.py --batch $b --layers 4,7,10 --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/b${b}_bn${bn}_u${un}_s${st}.json 2>> $OUT/err.log || continue
  python3 -c "
import json; d=json.load(open('$OUT/b${b}_bn${bn}_u${un}_s${st}.json')); pl=d['roofline']['per_layer']
print('b=$b bn=$bn u=$un stage=$st', [l['us_per_forward'][2] for l in pl])"
done; done; done; done
