#!/bin/bash
# bench (kernels only) + ncu --set full of K0/K1/GEMM on the first 56x56 layer
# and the first 7x7 layer (launch indices from bench.py --layers).
set -u
OUT=gpurun_out/${1:-r2p}
KREGEX=${2:-"input_range|input_quant|gemm_epilogue"}
mkdir -p $OUT
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/bench.json 2> $OUT/bench.err
for L in 0 10; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KREGEX" -s 9 -c 3 \
    -o $OUT/prof_L$L python bench.py --layers $L --steps 1 --warmup 3 --no-cpu --no-e2e --no-verify > $OUT/ncu_L$L.log 2>&1
done
python3 - <<'PY'
import json,sys
d=json.loads(open("gpurun_out/%s/bench.json" % sys.argv[1] if len(sys.argv)>1 else "x").read())
PY
head -c 300 $OUT/bench.json; echo
python3 -c "
import json; d=json.loads(open('$OUT/bench.json').read())
print(d['value'], d['ms_per_step']); [print(l) for l in d['roofline']['per_layer']]"
