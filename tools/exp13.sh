#!/bin/bash
mkdir -p gpurun_out/exp13
o=gpurun_out/exp13
for rep in 1 2; do for v in sus0 sus10m sus1u; do
  timeout 300 python tools/gemm_ab.py abso/$v.so >> $o/gemm_ab.jsonl 2>&1
  timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | grep '^{' | sed "s/^/$v /" | cut -c1-110 >> $o/attn_ab.txt
done; done
cat $o/gemm_ab.jsonl; cat $o/attn_ab.txt
