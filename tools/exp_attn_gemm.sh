#!/bin/bash
# Round-2 experiments on one B200: attention forward variants (correctness + A/B
# timing), GEMM per-role wait trace, the cuBLAS kernels at the step's shapes.
mkdir -p gpurun_out/exp
o=gpurun_out/exp
for v in 1 3; do
  DPN_ATTN_FWD=$v timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -p no:cacheprovider > $o/attn_tests_v$v.log 2>&1; echo "v$v tests: $(tail -1 $o/attn_tests_v$v.log)"
  DPN_ATTN_FWD=$v timeout 300 python tools/attn_micro.py > $o/attn_micro_v$v.jsonl 2>&1; cat $o/attn_micro_v$v.jsonl | cut -c1-200
done
timeout 300 python tools/gemm_trace.py > $o/gemm_trace.txt 2>&1; cat $o/gemm_trace.txt
timeout 300 python tools/cublas_names.py > $o/cublas_names.txt 2>&1; cat $o/cublas_names.txt | cut -c1-200
