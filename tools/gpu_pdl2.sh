#!/bin/bash
# PDL (programmatic dependent launch) under CUDA-graph replay, per-GPU batches.
set -u
OUT=gpurun_out/${1:-pdl2}
mkdir -p $OUT
for b in 256 64 32; do for p in 0 1; do
  LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so LANCE_PDL=$p timeout 600 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/b${b}_p$p.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/b${b}_p$p.json'))
print('batch $b pdl $p', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'])"
done; done
