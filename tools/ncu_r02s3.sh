#!/bin/bash
# Round-2 (session 3) ncu evidence for the bench configuration (one GPU): launch
# list of one BERT-large b=64 step with m=8 micro-batches (the m=32 step's kernel
# mix at a quarter of the launches), full-set captures of the GEMM and attention.
mkdir -p gpurun_out
N="--nvtx --nvtx-include timed_step/"
timeout 1200 ncu $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02s3_launches_step.csv python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/r02s3_ncu_launch.log 2>&1
timeout 600 ncu $N --set full --clock-control none --import-source on -k regex:gemm_kernel -s 200 -c 4 -o gpurun_out/r02s3_prof_gemm -f python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/r02s3_ncu_gemm.log 2>&1
timeout 600 ncu $N --set full --clock-control none --import-source on -k regex:"attn_fwd_kernel|attn_bwd_kernel" -s 10 -c 2 -o gpurun_out/r02s3_prof_attn -f python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/r02s3_ncu_attn.log 2>&1
timeout 600 ncu $N --set full --clock-control none -k regex:"ln_bwd_fused|ln_fwd|adamw|xent|attn_dq_store" -s 40 -c 8 -o gpurun_out/r02s3_prof_hbm -f python tools/ncu_step.py bert-large 64 8 serial > gpurun_out/r02s3_ncu_hbm.log 2>&1
python tools/ncu_summary.py gpurun_out/r02s3_ncu_step_b64.md gpurun_out/r02s3_launches_step.csv gpurun_out/r02s3_prof_gemm.ncu-rep gpurun_out/r02s3_prof_attn.ncu-rep gpurun_out/r02s3_prof_hbm.ncu-rep > gpurun_out/r02s3_ncu_summary.log 2>&1
gzip -9 -f gpurun_out/r02s3_launches_step.csv
rm -f gpurun_out/r02s3_prof_hbm.ncu-rep
ls -la gpurun_out | tail -12
