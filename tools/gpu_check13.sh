#!/bin/bash
set -x
mkdir -p gpurun_out
for st in 1 2 4; do
  timeout 600 python bench.py --stages $st --micro-batches 32 --no-cpu-baseline > gpurun_out/bench_st$st.json 2> gpurun_out/bench_st$st.err
done
timeout 2400 python tools/max_batch.py --model gpt2-xl --stages 8 --cap-gib 40 --b-max 64 --out gpurun_out/maxbatch_gpt2.json > gpurun_out/maxbatch_gpt2.log 2>&1
