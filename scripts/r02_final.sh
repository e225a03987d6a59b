#!/bin/bash
# Round-2 final measurement pass (on the GPU box): every bench line, the
# reference arm, a 2-rank smoke of the multi-process bench path, the launch
# list of one step and ncu captures of the step's kernel classes.
set -u
OUT=${1:-gpurun_out/r2f}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt
timeout 1200 python bench.py --steps 5 --warmup 3 > $OUT/bench_llama2_7b_16k.json 2> $OUT/bench_llama2_7b_16k.err
for p in bf16 fp32; do
  timeout 1200 python bench.py --steps 5 --warmup 3 --scoring-precision $p --no-cpu --no-law \
      > $OUT/bench_llama2_7b_16k_$p.json 2> $OUT/bench_llama2_7b_16k_$p.err
done
for c in llama2_7b_4k llama2_7b_32k llama3_8b_16k mistral_7b_32k opt_6.7b_64k tiny; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --backend gloo --config llama2_7b_4k --steps 2 --warmup 3 \
    --no-dense --no-law --no-cpu --no-audit > $OUT/bench_2rank_gloo.json 2> $OUT/bench_2rank_gloo.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/launches.log 2>&1
cap() {  # tag regex skip count
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o $OUT/full_$1 \
      python scripts/profile_step.py > $OUT/full_$1.log 2>&1
}
cap gateup "EpiGateUpT<(\(bool\)0|false)>" 0 1
cap refine "EpiGateUpT<(\(bool\)1|true)>|mlp_token_band|mlp_patch_rows" 0 3
cap fwd "flash_fwd_kernel" 0 1
cap dkdv "flash_bwd_dkdv_kernel" 0 1
cap dq "flash_bwd_dq_kernel" 0 1
cap dX "Bound<256, lemo::EpiStoreF32>" 16 1
cap blockembed "block_embed_kernel" 0 1
ls $OUT
