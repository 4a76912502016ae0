#!/bin/bash
mkdir -p gpurun_out/exp3
o=gpurun_out/exp3
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py tests/test_parity_real_configs_gpu.py -q -x -p no:cacheprovider > $o/tests.log 2>&1; tail -3 $o/tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench_b48.json 2>$o/b48.err; tail -1 $o/bench_b48.json | cut -c1-200
for mb in 64 74; do
  timeout 600 python bench.py --micro-batch $mb --steps 3 --no-cpu-baseline > $o/bench_b$mb.json 2>$o/b$mb.err; tail -1 $o/bench_b$mb.json | cut -c1-200; tail -2 $o/b$mb.err
done
