#!/bin/bash
# Round-2 profile set (on the GPU box): launch list of one LeMo step and
# `ncu --set full` captures of the step's kernel classes.
set -u
OUT=${1:-gpurun_out/r2}
mkdir -p $OUT
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/launches.log 2>&1
cap() {  # tag regex skip count
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      --kernel-name-base demangled -k regex:"$2" -s $3 -c $4 -o $OUT/full_$1 \
      python scripts/profile_step.py > $OUT/full_$1.log 2>&1
}
cap gateup "EpiGateUp" 0 1
cap dX "Bound<256, lemo::EpiStoreF32>" 16 2
cap lmhead "Bound<256, lemo::EpiStoreF32>" 0 1
cap split3 "EpiSplit3" 0 3
cap f32exact "gemm_tn_kernel<64, lemo::Bound<64, lemo::EpiStoreF32>, false, 2>" 0 1
cap fwd "flash_fwd_kernel" 0 1
cap dkdv "flash_bwd_dkdv_kernel" 0 1
cap dq "flash_bwd_dq_kernel" 0 1
cap qkv "EpiQKV" 0 1
cap scatter "EpiScatterAdd" 0 1
cap dgateup "EpiDGateUp" 0 1
cap loragrads "lora_grads_kernel" 0 1
cap cerows "ce_rows_kernel" 0 1
cap compact "mlp_compact_kernel" 0 1
ls $OUT
