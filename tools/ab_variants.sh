#!/bin/bash
# Same-box A/B of library builds that differ only in build-time knobs (run on
# the GPU box after building the variants here with tools/build_variant.sh):
#   tools/build_variant.sh base
#   tools/build_variant.sh sus0 -DDPN_MBAR_SUSPEND_NS=0
#   gpurun -- 'bash tools/ab_variants.sh base sus0'
# Each variant runs twice, interleaved, through the GEMM, attention and
# LayerNorm micro-benchmarks; JSON lines land in gpurun_out/ab/.
# Knobs: DPN_GEMM_MAX_STAGES / DPN_GEMM_GROUP / DPN_GEMM_L2_PROMO / DPN_GEMM_HINT / DPN_GEMM_EPI_WARPS /
# DPN_GEMM_COMMIT_PAIRS
# (gemm.cu), DPN_MBAR_SUSPEND_NS (common.cuh), DPN_ATTN_POLY / DPN_ATTN_POLY_BWD /
# DPN_ATTN_PACK_ALU (attention.cu), DPN_LN_ROWS / DPN_LN_CTAS (kernels.cu).
mkdir -p gpurun_out/ab
for rep in 1 2; do for v in "$@"; do
  timeout 300 python tools/gemm_ab.py abso/$v.so >> gpurun_out/ab/gemm_ab.jsonl 2>&1
  timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | grep '^{' | sed "s/^/$v /" >> gpurun_out/ab/attn_ab.txt
  timeout 300 python tools/ln_ab.py abso/$v.so >> gpurun_out/ab/ln_ab.jsonl 2>&1
done; done
cat gpurun_out/ab/*
