#!/bin/bash
# GEMM decomposition experiments: LANCE_GEMM_EXP=1 (no epilogue math/stores),
# 2 (no MMAs), 3 (neither), and tile-width variants.  Layers 0 and 10.
set -u
TAG=${1:-exp}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CFG_LIST=${CFG_LIST:-"EXP=0;EXP=1;EXP=2;EXP=3;BN=64;BN=64 EXP=1;BN=16"}
IFS=';' read -ra CFGS <<< "$CFG_LIST"
for cfg in "${CFGS[@]}"; do
  envs=""
  for kv in $cfg; do envs="$envs LANCE_GEMM_$kv"; done
  echo "== $cfg" >> $OUT/exp.txt
  env $envs timeout 120 python bench.py --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
echo done
