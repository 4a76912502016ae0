#!/bin/bash
mkdir -p gpurun_out/exp10
o=gpurun_out/exp10
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -p no:cacheprovider > $o/tests.log 2>&1; echo "tests: $(tail -1 $o/tests.log)"
for rep in 1 2; do for v in poly0 poly1 poly2; do timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | grep '^{' | sed "s/^/$v /" | cut -c1-110 >> $o/attn_ab.txt; done; done; cat $o/attn_ab.txt
