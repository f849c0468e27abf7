#!/bin/bash
# The other BASELINE configs on the current build: config 4 (F(4x4)), config 2
# (VGG-16-CIFAR independent layers and the chained stack, F(2x2) and F(4x4)),
# config 3 with NCHW input.
set -u
OUT=gpurun_out/${1:-configs}
mkdir -p $OUT
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err;
  python3 -c "
import json; d=json.load(open('$OUT/$name.json')); print('$name', round(d['value']), round(d['ms_per_step'],4), (d.get('parity') or {}).get('bitexact'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; }
run f4 --tile-m 4 --steps 20 --warmup 5
run vgg --workload vgg16_cifar --steps 20 --warmup 5
run stack --workload vgg16_cifar --stack --steps 20 --warmup 5 --no-cpu
run stack_f4 --workload vgg16_cifar --stack --tile-m 4 --steps 20 --warmup 5 --no-cpu
run nchw --layout nchw --steps 20 --warmup 5 --no-cpu --no-e2e
