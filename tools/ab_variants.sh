#!/bin/bash
# Build variant libraries of one translation unit with extra -D flags and link
# them with the rest of the current build:  tools/ab_variants.sh <src.cu> TAG:"-DX=1 -DY=2" ...
# -> scratch/ab_TAG/liblance_b200.so (LANCE_LIB_PATH selects one at run time).
set -e
SRC=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null
B=paper_2003_08646_b200/_build
base=$(basename $SRC .cu)
for spec in "$@"; do
  tag=${spec%%:*}; defs=${spec#*:}
  D=scratch/ab_$tag; mkdir -p $D
  nvcc -DLANCE_JMAJOR=0 $defs -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -c paper_2003_08646_b200/csrc/$SRC -o $D/$base.o
  objs=$(ls $B/*.o | grep -v "/$base.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/liblance_b200.so $objs $D/$base.o
  echo built $D
done
