#!/bin/bash
# ncu --set full captures of the hot kernels (one GPU, short commands).
#   gpurun --timeout 1800 -- bash tools/profile.sh <tag> [layer ...]
set -u
TAG=${1:-prof}; shift
LAYERS=${@:-0 10}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
[ -x scratch/umma_bench ] && timeout 60 scratch/umma_bench > $OUT/umma_bench.txt 2>&1
for L in $LAYERS; do
  for K in input_range input_quant gemm_epilogue; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o $OUT/${K}_L$L python bench.py --layers $L --steps 1 --warmup 3 --no-cpu --no-e2e \
      > $OUT/ncu_${K}_L$L.log 2>&1
  done
done
echo done
