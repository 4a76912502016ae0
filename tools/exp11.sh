#!/bin/bash
mkdir -p gpurun_out/exp11
o=gpurun_out/exp11
for rep in 1 2; do for v in h0 h1 h2; do timeout 300 python tools/gemm_ab.py abso/$v.so >> $o/gemm_ab.jsonl 2>&1; done; done; cat $o/gemm_ab.jsonl
