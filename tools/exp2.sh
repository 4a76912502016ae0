#!/bin/bash
mkdir -p gpurun_out/exp2
o=gpurun_out/exp2
for v in 3 1; do
  DPN_ATTN_FWD=$v timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -p no:cacheprovider > $o/attn_tests_v$v.log 2>&1; echo "v$v tests: $(tail -1 $o/attn_tests_v$v.log)"
  DPN_ATTN_FWD=$v timeout 300 python tools/attn_micro.py > $o/attn_micro_v$v.jsonl 2>&1; cut -c1-120 $o/attn_micro_v$v.jsonl
done
for rep in 1 2; do for v in base st4 g16 g4 p128; do
  timeout 300 python tools/gemm_ab.py abso/$v.so >> $o/gemm_ab.jsonl 2>&1
done; done
cat $o/gemm_ab.jsonl
