#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or layernorm or xent" > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 300 python tools/attn_micro.py > gpurun_out/attn_micro.txt 2>&1
timeout 600 python tools/profile_step.py bert-large 32 32 serial > gpurun_out/breakdown_b32.txt 2>&1
