#!/bin/bash
set -u
OUT=gpurun_out/${1:-r2h}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_stack.py tests/test_gpu_nchw.py tests/test_gpu_large.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash tools/gpu_ab.sh ${1:-r2h}_ab
