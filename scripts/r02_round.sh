#!/bin/bash
# Round-2 GPU pass: tests, default bench (+ reference arm optional), all configs.
OUT=${1:-gpurun_out/r2c}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $OUT/bench_llama2_7b_16k.json 2> $OUT/bench_llama2_7b_16k.err
tail -c 400 $OUT/bench_llama2_7b_16k.json; echo
for c in llama2_7b_4k llama2_7b_32k llama3_8b_16k mistral_7b_32k opt_6.7b_64k tiny; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
ls $OUT
