#!/bin/bash
# A/B of library variants (scratch/ab_*/liblance_b200.so vs the in-tree build),
# interleaved twice; kernel-only bench lines.  Usage: gpu_ab.sh OUT [extra bench args]
set -u
OUT=gpurun_out/${1:-ab}; shift
mkdir -p $OUT
for rep in 1 2; do
  for v in main scratch/ab_*; do
    n=$(basename $v)
    if [ "$v" = main ]; then lib=paper_2003_08646_b200/_build/liblance_b200.so; else lib=$v/liblance_b200.so; fi
    LANCE_LIB_PATH=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e "$@" > $OUT/bench_${n}_$rep.json 2>> $OUT/err.log
    python3 -c "
import json; d=json.load(open('$OUT/bench_${n}_$rep.json')); pl=d['roofline']['per_layer']
print('$n', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'] if d.get('parity') else None, [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
  done
done
