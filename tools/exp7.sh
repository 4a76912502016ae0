#!/bin/bash
mkdir -p gpurun_out/exp7
o=gpurun_out/exp7
timeout 400 python -m pytest tests/test_kernels_gpu.py -q -k "layernorm or attention" -p no:cacheprovider > $o/tests.log 2>&1; echo "tests: $(tail -1 $o/tests.log)"
for rep in 1 2; do for v in base ln_r2d3 ln_r1d4c3 ln_r1d6; do timeout 300 python tools/ln_ab.py abso/$v.so >> $o/ln_ab.jsonl 2>&1; done; done; cat $o/ln_ab.jsonl
timeout 600 python bench.py --no-cpu-baseline --steps 4 > $o/bench_b64.json 2>$o/b64.err; tail -1 $o/bench_b64.json | cut -c1-200
