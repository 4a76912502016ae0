#!/bin/bash
mkdir -p gpurun_out/exp5
o=gpurun_out/exp5
timeout 400 python -m pytest tests/test_kernels_gpu.py tests/test_cnn_kernels_gpu.py -q -p no:cacheprovider > $o/tests.log 2>&1; echo "tests: $(tail -1 $o/tests.log)"
for v in base sts base sts; do timeout 300 python tools/gemm_ab.py abso/$v.so >> $o/gemm_ab.jsonl 2>&1; done; cat $o/gemm_ab.jsonl
for v in qdb sts qdb sts; do timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | sed "s/^/$v /" | cut -c1-110 >> $o/attn_ab.txt; done; cat $o/attn_ab.txt
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench_b64.json 2>$o/b64.err; tail -1 $o/bench_b64.json | cut -c1-200
