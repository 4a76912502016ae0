#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pipeline_gpu.py -k sync -x -q > gpurun_out/pytest_sync.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sync.log
timeout 300 python tools/gemm_breakdown.py > gpurun_out/gemm_breakdown.txt 2>&1
timeout 300 python tools/gemm_micro.py > gpurun_out/gemm_micro.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1500 -c 6 -o gpurun_out/prof_gemm python tools/ncu_target.py > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 300 -c 4 -o gpurun_out/prof_attn python tools/ncu_target.py > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"adamw|ln_|colred|xent" -s 400 -c 8 -o gpurun_out/prof_hbm python tools/ncu_target.py > gpurun_out/ncu_hbm.log 2>&1
ls -la gpurun_out
