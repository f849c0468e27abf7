#!/bin/bash
# F(4x4) GEMM experiments: env configurations (CFG_LIST, ';'-separated, each a
# space-separated list of LANCE_F4_* assignments) on layers 0, 4, 7, 10.
set -u
TAG=${1:-f4exp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CFG_LIST=${CFG_LIST:-"LANES=1;LANES=2;LANES=4"}
IFS=';' read -ra CFGS <<< "$CFG_LIST"
for cfg in "${CFGS[@]}"; do
  envs=""
  for kv in $cfg; do envs="$envs LANCE_F4_$kv"; done
  echo "== $cfg" >> $OUT/exp.txt
  env $envs timeout 120 python bench.py --tile-m 4 --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
echo done
