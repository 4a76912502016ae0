#!/bin/bash
# Quick GPU re-check after a kernel change: kernel + pipeline + real-config parity tests, default bench.
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py tests/test_parity_real_configs_gpu.py tests/test_cuda_graph_gpu.py -q -p no:cacheprovider > gpurun_out/quick/tests.log 2>&1; tail -2 gpurun_out/quick/tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 4 > gpurun_out/quick/bench.json 2>gpurun_out/quick/bench.err; tail -1 gpurun_out/quick/bench.json | cut -c1-160
