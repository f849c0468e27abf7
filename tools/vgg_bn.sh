OUT=gpurun_out/vggbn; mkdir -p $OUT
for cfg in "" "LANCE_GEMM_BN=32" "LANCE_GEMM_BN=16"; do
  echo "== $cfg" >> $OUT/exp.txt
  env $cfg timeout 120 python bench.py --workload vgg16_cifar --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/b.json 2>> $OUT/exp.err
  python -c "
import json; d=json.load(open('$OUT/b.json')); print('  value', round(d['value']))
for l in d['roofline']['per_layer']: print('  ', l['c'], l['k'], l['h'], l['us_per_forward'])" >> $OUT/exp.txt
done
