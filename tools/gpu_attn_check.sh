#!/bin/bash
# Attention kernel tests + micro-benchmark + bench after an attention change.
mkdir -p gpurun_out/attn_check
o=gpurun_out/attn_check
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k "attention" -p no:cacheprovider > $o/tests.log 2>&1; echo "tests: $(tail -1 $o/tests.log)"
timeout 300 python tools/attn_micro.py 2>&1 | grep '^{' | cut -c1-130 | tee $o/attn_micro.txt
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench.json 2>$o/bench.err; tail -1 $o/bench.json | cut -c1-160
