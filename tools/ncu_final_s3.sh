#!/bin/bash
# Full-set ncu captures of the final code's GEMM and attention backward inside the
# bench step (b=64, m=8), summarised into a markdown file.
mkdir -p gpurun_out
N="--nvtx --nvtx-include timed_step/"
timeout 600 ncu $N --set full --clock-control none --import-source on -k regex:gemm_kernel -s 200 -c 4 -o gpurun_out/s3f_prof_gemm -f python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/s3f_ncu_gemm.log 2>&1
timeout 600 ncu $N --set full --clock-control none --import-source on -k regex:"attn_bwd_kernel" -s 4 -c 1 -o gpurun_out/s3f_prof_attn_bwd -f python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/s3f_ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/r02s3_final_ncu.md gpurun_out/s3f_prof_gemm.ncu-rep gpurun_out/s3f_prof_attn_bwd.ncu-rep > gpurun_out/s3f_summary.log 2>&1
ls -la gpurun_out | grep s3f
