#!/bin/bash
# ncu --set full with source correlation of the attention kernels at the bench shape
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd|attn_bwd_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_attn_r02 -f python tools/attn_one.py > gpurun_out/ncu_attn.log 2>&1
ncu -i gpurun_out/prof_attn_r02.ncu-rep --page source --csv --print-source sass -k regex:attn_fwd > gpurun_out/attn_fwd_source.csv 2>/dev/null
ncu -i gpurun_out/prof_attn_r02.ncu-rep --page raw --csv > gpurun_out/attn_raw.csv 2>/dev/null
ls -la gpurun_out/prof_attn_r02.ncu-rep
