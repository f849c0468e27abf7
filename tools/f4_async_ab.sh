OUT=gpurun_out/f4as; mkdir -p $OUT
LANCE_F4_ASYNC=2 timeout 300 python -m pytest tests/test_gpu_f4.py -x -q > $OUT/t2.log 2>&1; echo rc=$? >> $OUT/t2.log
LANCE_F4_ASYNC=4 timeout 300 python -m pytest tests/test_gpu_f4.py -x -q > $OUT/t4.log 2>&1; echo rc=$? >> $OUT/t4.log
for rep in 1 2; do
for cfg in "" "LANCE_F4_ASYNC=2" "LANCE_F4_ASYNC=4"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --tile-m 4 --layers 0,4,7,10 --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json'))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
done
