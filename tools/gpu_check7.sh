#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --micro-batch 16 --no-cpu-baseline > gpurun_out/bench_b16.json 2> gpurun_out/bench_b16.err
timeout 900 python bench.py --micro-batch 32 --no-cpu-baseline > gpurun_out/bench_b32.json 2> gpurun_out/bench_b32.err
timeout 300 python tools/profile_step.py amoebanet-d 64 32 > gpurun_out/breakdown_amoeba.txt 2>&1
