#!/bin/bash
mkdir -p gpurun_out/exp4
o=gpurun_out/exp4
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -p no:cacheprovider > $o/attn_tests.log 2>&1; echo "tests: $(tail -1 $o/attn_tests.log)"
for v in base qdb base qdb; do
  timeout 300 python tools/attn_micro.py abso/$v.so 2>&1 | sed "s/^/$v /" | cut -c1-110 >> $o/attn_ab.txt
done
cat $o/attn_ab.txt
