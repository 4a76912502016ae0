#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python tools/max_batch.py --model amoebanet-d --stages 8 --cap-gib 40 --b-max 1024 --out gpurun_out/maxbatch_amoeba.json > gpurun_out/maxbatch_amoeba.log 2>&1
timeout 900 python bench.py --model t5-large --stages 4 --micro-batch 16 --micro-batches 16 --no-cpu-baseline > gpurun_out/bench_t5_4stage.json 2> gpurun_out/bench_t5_4stage.err
