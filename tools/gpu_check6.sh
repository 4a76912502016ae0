#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --model t5-large --micro-batch 16 --no-cpu-baseline > gpurun_out/bench_t5.json 2> gpurun_out/bench_t5.err
timeout 900 python bench.py --model amoebanet-d --micro-batch 64 --no-cpu-baseline > gpurun_out/bench_amoeba.json 2> gpurun_out/bench_amoeba.err
timeout 900 python bench.py --model gpt2-xl --micro-batch 4 --no-cpu-baseline > gpurun_out/bench_gpt2.json 2> gpurun_out/bench_gpt2.err
