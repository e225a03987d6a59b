#!/bin/bash
# Round-2 bench lines for every BASELINE config + the missing ncu rows.
OUT=${1:-gpurun_out/r2b}
mkdir -p $OUT
for c in llama2_7b_4k llama2_7b_32k llama3_8b_16k mistral_7b_32k opt_6.7b_64k tiny; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  tail -c 300 $OUT/bench_$c.json; echo
done
cap() {  # tag regex skip count
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o $OUT/full_$1 \
      python scripts/profile_step.py > $OUT/full_$1.log 2>&1
}
cap dX "EpiStoreF32>>" 16 2
cap lmhead "EpiStoreF32>>" 0 1
cap f32exact "EpiStoreF32>, \(bool\)0, \(int\)2>" 0 1
ls $OUT
