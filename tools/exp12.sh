#!/bin/bash
mkdir -p gpurun_out/exp12
o=gpurun_out/exp12
for v in 4 1; do
  DPN_ATTN_FWD=$v timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -p no:cacheprovider > $o/tests_v$v.log 2>&1; echo "v$v tests: $(tail -1 $o/tests_v$v.log)"
done
for rep in 1 2; do for v in 1 4; do DPN_ATTN_FWD=$v timeout 300 python tools/attn_micro.py 2>&1 | grep '^{' | sed "s/^/v$v /" | cut -c1-110 >> $o/attn_ab.txt; done; done; cat $o/attn_ab.txt
