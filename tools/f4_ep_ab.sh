OUT=gpurun_out/f4ep; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_f4.py tests/test_gpu_stack.py -x -q > $OUT/t.log 2>&1; echo rc=$? >> $OUT/t.log
for rep in 1 2; do
  timeout 120 python bench.py --tile-m 4 --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
