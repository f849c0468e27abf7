#!/bin/bash
# The N>1 bench path on a 1-GPU lease: --gpus 2 spawns 2 ranks (both on the one
# device: a logic check of spawn / strong split / NCCL verify / max-over-ranks,
# not a scaling number), per-shard and global-fit modes.
set -u
OUT=gpurun_out/${1:-multi}
mkdir -p $OUT
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/g2.json 2> $OUT/g2.err; echo "rc=$?"
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu --mode global > $OUT/g2_global.json 2> $OUT/g2_global.err; echo "rc=$?"
for f in g2 g2_global; do python3 -c "
import json; d=json.load(open('$OUT/$f.json')); print('$f', d['n_gpus'], round(d['value']), d['ms_per_step'], d['config'].get('parallelism'), d.get('parity'), d.get('verify_sharded'))" || tail -5 $OUT/$f.err; done
grep -i "nccl\|rank" $OUT/g2.err | head -5
