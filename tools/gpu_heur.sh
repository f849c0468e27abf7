#!/bin/bash
set -u
OUT=gpurun_out/${1:-heur}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_stack.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
for v in main ab_oldheur; do
  if [ $v = main ]; then lib=paper_2003_08646_b200/_build/liblance_b200.so; else lib=scratch/$v/liblance_b200.so; fi
  for b in 256 128 64 32; do
    LANCE_LIB_PATH=$lib timeout 600 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/${v}_b$b.json 2>> $OUT/err.log
    python3 -c "
import json; d=json.load(open('$OUT/${v}_b$b.json')); pl=d['roofline']['per_layer']
print('$v batch $b', round(d['value']), round(d['ms_per_step'],4), [pl[i]['us_per_forward'][2] for i in (0,4,7,10)])"
  done
  LANCE_LIB_PATH=$lib timeout 600 python bench.py --workload vgg16_cifar --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify > $OUT/${v}_vgg.json 2>> $OUT/err.log
  LANCE_LIB_PATH=$lib timeout 600 python bench.py --workload vgg16_cifar --stack --steps 20 --warmup 5 --no-cpu --no-e2e > $OUT/${v}_stack.json 2>> $OUT/err.log
  python3 -c "
import json
for w in ('vgg','stack'):
  d=json.load(open('$OUT/${v}_'+w+'.json')); print('$v', w, round(d['value']), round(d['ms_per_step'],4))"
done
