#!/bin/bash
# ncu evidence for the bench configuration (one GPU): launch list of one step,
# full-set captures of the top kernels.
set -x
mkdir -p gpurun_out
N="--nvtx --nvtx-include timed_step/"
timeout 1500 ncu $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/ncu_step.py bert-large 32 32 serial > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu $N --set full --clock-control none --import-source on -k regex:gemm_kernel -s 200 -c 6 -o gpurun_out/prof_gemm python tools/ncu_step.py bert-large 32 32 serial > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu $N --set full --clock-control none --import-source on -k regex:attn_ -s 20 -c 6 -o gpurun_out/prof_attn python tools/ncu_step.py bert-large 32 32 serial > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu $N --set full --clock-control none -k regex:"adamw|ln_|colred|xent" -s 100 -c 10 -o gpurun_out/prof_hbm python tools/ncu_step.py bert-large 32 32 serial > gpurun_out/ncu_hbm.log 2>&1
timeout 600 ncu $N --set full --clock-control none -k regex:"xent" -c 1 -o gpurun_out/prof_xent python tools/ncu_step.py bert-large 32 32 serial > gpurun_out/ncu_xent.log 2>&1
# summarise on the box (gpurun copies back at most 64 MiB): keep the GEMM report only
python tools/ncu_summary.py gpurun_out/ncu_step_b32.md gpurun_out/launches_step.csv gpurun_out/prof_gemm.ncu-rep gpurun_out/prof_attn.ncu-rep gpurun_out/prof_hbm.ncu-rep gpurun_out/prof_xent.ncu-rep > gpurun_out/ncu_summary.log 2>&1
gzip -9 gpurun_out/launches_step.csv
rm -f gpurun_out/prof_attn.ncu-rep gpurun_out/prof_hbm.ncu-rep gpurun_out/prof_xent.ncu-rep
ls -la gpurun_out
