#!/bin/bash
# full-set ncu of the HBM-bound step kernels (xent, column reductions) at the bench shape
set -x
mkdir -p gpurun_out
N="--nvtx --nvtx-include timed_step/"
timeout 900 ncu $N --set full --clock-control none --import-source on -k regex:"xent|colred" -s 4 -c 6 -o gpurun_out/prof_small python tools/ncu_step.py bert-large 32 32 serial > gpurun_out/ncu_small.log 2>&1
