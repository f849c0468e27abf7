#!/bin/bash
# ncu --set full of the GEMM under an experiment switch, one layer.
set -u
TAG=$1; EXPV=$2; L=$3
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
LANCE_GEMM_EXP=$EXPV timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_epilogue -s 3 -c 1 \
    -o $OUT/gemm_e${EXPV}_L$L python bench.py --layers $L --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_e${EXPV}_L$L.log 2>&1
echo done
