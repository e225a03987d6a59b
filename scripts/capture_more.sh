#!/bin/bash
# Extra ncu --set full captures for the per-kernel roofline table.
OUT=${1:-gpurun_out/r1e}
mkdir -p $OUT
cap() {  # tag regex skip count
  timeout 600 ncu --profile-from-start off --set full --clock-control none --kernel-name-base demangled \
      -k regex:"$2" -s $3 -c $4 -o $OUT/full_$1 python scripts/profile_step.py > $OUT/full_$1.log 2>&1
}
cap dX "Bound<256, lemo::EpiStoreF32>" 16 2
cap lmhead "Bound<256, lemo::EpiStoreF32>" 0 2
cap select "select_kernel" 0 1
cap colsum "colsum_clamped_kernel" 0 1
cap mlpscores "mlp_block_scores_warp_kernel" 0 1
cap gatherrms "gather_rmsnorm_kernel" 1 1
cap cerows "ce_rows_kernel" 0 1
cap split3 "EpiSplit3" 0 1
cap gatherrows "gather_rows_bf16_kernel" 0 1
cap dO "EpiStoreBF16" 0 1
ls $OUT
