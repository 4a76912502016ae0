#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python tools/max_batch.py --model t5-large --stages 8 --cap-gib 40 --b-max 256 --out gpurun_out/maxbatch_t5.json > gpurun_out/maxbatch_t5.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
