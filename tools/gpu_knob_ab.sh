#!/bin/bash
# Interleaved A/B of one LANCE_* knob (profiling library): gpu_knob_ab.sh OUT NAME V1 V2 [bench args]
set -u
OUT=gpurun_out/$1; NAME=$2; V1=$3; V2=$4; shift 4
mkdir -p $OUT
for rep in 1 2; do for v in $V1 $V2; do
  env LANCE_LIB_PATH=scratch/ab_prof/liblance_b200.so $NAME=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e "$@" > $OUT/${v}_$rep.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/${v}_$rep.json')); pl=d['roofline']['per_layer']
print('$NAME=$v', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'] if d.get('parity') else None, [pl[i]['us_per_forward'] for i in (0,4,7,10) if i < len(pl)])"
done; done
