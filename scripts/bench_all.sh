set -u
mkdir -p gpurun_out/${OUT:-b9}
timeout 400 python bench.py > gpurun_out/${OUT:-b9}/llama2_7b_16k.json 2> gpurun_out/${OUT:-b9}/llama2_7b_16k.err
for c in llama2_7b_32k llama3_8b_16k mistral_7b_32k opt_6.7b_64k llama2_7b_4k tiny; do
  timeout 500 python bench.py --config $c --no-cpu > gpurun_out/${OUT:-b9}/$c.json 2> gpurun_out/${OUT:-b9}/$c.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${OUT:-b9}/reference.json 2> gpurun_out/${OUT:-b9}/reference.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${OUT:-b9}/launches.csv python scripts/profile_step.py > gpurun_out/${OUT:-b9}/launches.log 2>&1
ls -la gpurun_out/${OUT:-b9}
# one ncu --set full capture per hot kernel of the step (summaries -> profiles/)
KERNELS="EpiGateUp EpiStoreF32 EpiScatterAdd flash_fwd_kernel flash_bwd_dkdv_kernel flash_bwd_dq_kernel" \
  NO_LAUNCHES=1 bash scripts/capture_profiles.sh gpurun_out/${OUT:-b9}/ncu > /dev/null 2>&1
ls gpurun_out/${OUT:-b9}/ncu
