#!/bin/bash
# Round-2 ncu evidence for the bench configuration (one GPU): launch list of one
# BERT-large b=32 step with m=8 micro-batches (the m=32 step's kernel mix at a
# quarter of the launches), and full-set captures of the GEMM and the fused
# LayerNorm backward.
mkdir -p gpurun_out
N="--nvtx --nvtx-include timed_step/"
timeout 1200 ncu $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_step.csv python tools/ncu_step.py bert-large 32 8 serial > gpurun_out/r02_ncu_launch.log 2>&1
timeout 600 ncu $N --set full --clock-control none --import-source on -k regex:gemm_kernel -s 200 -c 4 -o gpurun_out/r02_prof_gemm -f python tools/ncu_step.py bert-large 32 8 serial > gpurun_out/r02_ncu_gemm.log 2>&1
timeout 600 ncu $N --set full --clock-control none -k regex:"ln_bwd_fused|ln_fwd|colred|adamw|xent" -s 40 -c 8 -o gpurun_out/r02_prof_hbm -f python tools/ncu_step.py bert-large 32 8 serial > gpurun_out/r02_ncu_hbm.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_step_b32.md gpurun_out/r02_launches_step.csv gpurun_out/r02_prof_gemm.ncu-rep gpurun_out/prof_attn_r02.ncu-rep gpurun_out/r02_prof_hbm.ncu-rep > gpurun_out/r02_ncu_summary.log 2>&1
gzip -9 -f gpurun_out/r02_launches_step.csv
rm -f gpurun_out/r02_prof_hbm.ncu-rep
ls -la gpurun_out | tail -20
