#!/bin/bash
mkdir -p gpurun_out/exp6
o=gpurun_out/exp6
timeout 400 python -m pytest tests/test_kernels_gpu.py -q -k "attention or layernorm" -p no:cacheprovider > $o/tests.log 2>&1; echo "tests: $(tail -1 $o/tests.log)"
for v in sts kvdb sts kvdb; do timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | sed "s/^/$v /" | cut -c1-110 >> $o/attn_ab.txt; done; cat $o/attn_ab.txt
for v in base kvdb base kvdb; do timeout 300 python tools/ln_ab.py abso/$v.so >> $o/ln_ab.jsonl 2>&1; done; cat $o/ln_ab.jsonl
