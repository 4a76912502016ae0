#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_cli.py -k "t5 or cli" -x -q > gpurun_out/pytest_t5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_t5.log
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size,launch__shared_mem_per_block --csv python tools/cublas_names.py > gpurun_out/cublas_names.csv 2>&1
