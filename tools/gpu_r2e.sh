#!/bin/bash
set -u
OUT=gpurun_out/r2e
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_nchw.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
bash tools/gpu_ab.sh r2e_ab
timeout 600 python bench.py --workload vgg16_cifar --stack --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/bench_stack.json 2> $OUT/bench_stack.err
python3 -c "
import json; d=json.load(open('$OUT/bench_stack.json')); print('stack', round(d['value']), round(d['ms_per_step'],4), d.get('parity'))"
tail -3 $OUT/bench_stack.err
