#!/bin/bash
set -u
OUT=gpurun_out/${1:-large}
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_large.py -x -q --durations 10 > $OUT/pytest_large.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_large.log
tail -12 $OUT/pytest_large.log
