#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/pytest_attn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_attn.log
timeout 300 python tools/attn_micro.py > gpurun_out/attn_micro.txt 2>&1
timeout 1800 python tools/max_batch.py --model amoebanet-d --stages 8 --cap-gib 40 --b-max 1024 --out gpurun_out/maxbatch_amoeba.json > gpurun_out/maxbatch_amoeba.log 2>&1
