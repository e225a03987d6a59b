#!/bin/bash
# Round-2 closing pass (GPU box): the headline bench line, its launch list and
# the full GPU test suite + smoke on the final code.
set -u
OUT=${1:-gpurun_out/r2g}
mkdir -p $OUT
timeout 1200 python bench.py --steps 5 --warmup 3 > $OUT/bench_llama2_7b_16k.json 2> $OUT/bench_llama2_7b_16k.err
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/launches.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
ls $OUT
