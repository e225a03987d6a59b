set -u
mkdir -p gpurun_out/b8
timeout 400 python bench.py > gpurun_out/b8/llama2_7b_16k.json 2> gpurun_out/b8/llama2_7b_16k.err
for c in llama2_7b_32k llama3_8b_16k mistral_7b_32k opt_6.7b_64k llama2_7b_4k; do
  timeout 500 python bench.py --config $c --no-cpu > gpurun_out/b8/$c.json 2> gpurun_out/b8/$c.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b8/reference.json 2> gpurun_out/b8/reference.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b8/launches.csv python scripts/profile_step.py > gpurun_out/b8/launches.log 2>&1
ls -la gpurun_out/b8
