#!/bin/bash
mkdir -p gpurun_out/exp9
o=gpurun_out/exp9
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py tests/test_parity_real_configs_gpu.py tests/test_abi.py -q -p no:cacheprovider > $o/tests.log 2>&1; tail -3 $o/tests.log
for v in kvdb spec kvdb spec; do timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | sed "s/^/$v /" | cut -c1-110 >> $o/attn_ab.txt; done; cat $o/attn_ab.txt
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench_b64.json 2>$o/b64.err; tail -1 $o/bench_b64.json | cut -c1-200
