#!/bin/bash
# On the GPU box: launch list of one training step + one `ncu --set full`
# capture per hot kernel (first instance inside the profiled step).
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
if [ -z "${NO_LAUNCHES:-}" ]; then
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/launches.log 2>&1
fi
KERNELS=${KERNELS:-"EpiGateUp EpiScatterAdd EpiQKV EpiDGateUp EpiStoreF32 flash_fwd_kernel flash_bwd_dkdv_kernel flash_bwd_dq_kernel block_embed_kernel rmsnorm_bwd_vec mlp_compact qkv_grad_prep lora_grads_kernel"}
for k in $KERNELS; do
  tag=$(echo $k | tr -cd 'A-Za-z0-9_')
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k regex:"$k" -c 1 -o $OUT/full_$tag python scripts/profile_step.py > $OUT/full_$tag.log 2>&1
done
ls $OUT
