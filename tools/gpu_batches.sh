#!/bin/bash
# Per-GPU batch sweep: the strong-scaling split gives 256/N images per GPU
# (N = 1, 2, 4, 8 -> 256, 128, 64, 32); one GPU at each per-rank batch,
# eager launches vs one CUDA graph per step.
set -u
OUT=gpurun_out/${1:-batches}
mkdir -p $OUT
shift || true
for b in 256 128 64 32; do for gr in 0 1; do
  timeout 600 python bench.py --batch $b --graph $gr --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify "$@" > $OUT/b${b}_g$gr.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/b${b}_g$gr.json')); pl=d['roofline']['per_layer']
print('batch $b graph $gr', round(d['value']), round(d['ms_per_step'],4), [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
done; done
