#!/bin/bash
# bench.py N=1 line (with parity + CPU baseline), spawn path at --gpus 2 (ranks
# share the one GPU over gloo: logic check only), new GPU tests.
set -u
OUT=gpurun_out/${1:-r2b}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ranges or shape or large_k" > $OUT/pytest_new.log 2>&1; echo "rc=$?" >> $OUT/pytest_new.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > $OUT/bench_g2.json 2> $OUT/bench_g2.err
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --mode global --no-verify > $OUT/bench_g2_global.json 2> $OUT/bench_g2_global.err
tail -2 $OUT/pytest_new.log; for f in $OUT/bench*.json; do echo == $f; head -c 400 $f; echo; done; tail -5 $OUT/*.err
