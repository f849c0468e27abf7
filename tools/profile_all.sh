#!/bin/bash
# ncu --set full captures of the current K0 / K1 / GEMM kernels (layer 0 = R64)
# and the GEMM on layer 10 (R512); one GPU, short commands.
set -u
TAG=$1
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() {  # name regex skip layer
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $OUT/$1 python bench.py --layers $4 --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_$1.log 2>&1
}
run k0_L0 input_range 3 0
run k1_L0 input_quant 3 0
run gemm_L0 gemm_epilogue 3 0
run gemm_L10 gemm_epilogue 3 10
run k1_L10 input_quant 3 10
echo done
