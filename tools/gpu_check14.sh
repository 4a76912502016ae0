#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python tools/max_batch.py --model t5-large --stages 8 --cap-gib 40 --b-max 128 --out gpurun_out/maxbatch_t5.json > gpurun_out/maxbatch_t5.log 2>&1
timeout 2400 python tools/max_batch.py --model gpt2-xl --stages 8 --cap-gib 40 --b-max 48 --out gpurun_out/maxbatch_gpt2.json > gpurun_out/maxbatch_gpt2.log 2>&1
