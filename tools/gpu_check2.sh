#!/bin/bash
# GEMM / F(4x4) parity suites + bench lines (F(2x2) twice, F(4x4), VGG stack).
set -u
OUT=gpurun_out/${1:-chk}
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_jsplit.py tests/test_gpu_f4.py tests/test_gpu_stack.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for r in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/f2_$r.json 2>> $OUT/err.log
  python3 -c "
import json; d=json.load(open('$OUT/f2_$r.json')); pl=d['roofline']['per_layer']
print('f2', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
done
timeout 600 python bench.py --tile-m 4 --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/f4.json 2>> $OUT/err.log
python3 -c "
import json; d=json.load(open('$OUT/f4.json')); pl=d['roofline']['per_layer']
print('f4', round(d['value']), round(d['ms_per_step'],4), d['parity']['bitexact'], [pl[i]['us_per_forward'] for i in (0,4,7,10)])"
timeout 600 python bench.py --workload vgg16_cifar --stack --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/stack.json 2>> $OUT/err.log
python3 -c "
import json; d=json.load(open('$OUT/stack.json')); print('stack', round(d['value']), round(d['ms_per_step'],4))"
