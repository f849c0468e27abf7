#!/bin/bash
# Per-GPU batch sweep: the strong-scaling split gives 256/N images per GPU
# (N = 1, 2, 4, 8 -> 256, 128, 64, 32); one GPU at each per-rank batch.
set -u
OUT=gpurun_out/${1:-batches}
mkdir -p $OUT
for b in 256 128 64 32; do
  timeout 600 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/b${b}.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/b${b}.json')); pl=d['roofline']['per_layer']
print('batch $b', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
done
