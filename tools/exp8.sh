#!/bin/bash
mkdir -p gpurun_out/exp8
o=gpurun_out/exp8
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py tests/test_parity_real_configs_gpu.py tests/test_abi.py -q -x -p no:cacheprovider > $o/tests.log 2>&1; tail -3 $o/tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench_b64.json 2>$o/b64.err; tail -1 $o/bench_b64.json | cut -c1-200
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench_b64_2.json 2>$o/b64_2.err; tail -1 $o/bench_b64_2.json | cut -c1-200
