#!/bin/bash
# GPU parity (GEMM-heavy suites) + interleaved A/B of scratch/ab_* vs the in-tree build.
set -u
OUT=gpurun_out/${1:-abt}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_jsplit.py tests/test_gpu_stack.py tests/test_gpu_large.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash tools/gpu_ab.sh ${1:-abt}_ab
