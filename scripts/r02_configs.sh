#!/bin/bash
# Bench lines of the non-headline BASELINE configs on the final code.
set -u
OUT=${1:-gpurun_out/r2i}
mkdir -p $OUT
for c in llama2_7b_4k llama2_7b_32k llama3_8b_16k mistral_7b_32k opt_6.7b_64k tiny; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
ls $OUT
