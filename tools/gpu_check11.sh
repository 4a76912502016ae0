#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --micro-batch 8 --no-cpu-baseline > gpurun_out/bench_b8.json 2> gpurun_out/bench_b8.err
timeout 600 python bench.py --model t5-large --micro-batch 16 --no-cpu-baseline > gpurun_out/bench_t5.json 2> gpurun_out/bench_t5.err
timeout 900 python bench.py --model gpt2-xl --micro-batch 4 --no-cpu-baseline > gpurun_out/bench_gpt2.json 2> gpurun_out/bench_gpt2.err
timeout 900 python bench.py --model amoebanet-d --micro-batch 64 --no-cpu-baseline > gpurun_out/bench_amoeba.json 2> gpurun_out/bench_amoeba.err
