#!/bin/bash
# Max-batch re-measurement on one B200 (tools/max_batch.py per model).
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_maxbatch.py -q > gpurun_out/pytest_maxbatch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_maxbatch.log
for m in ${MODELS:-t5-large gpt2-xl}; do
  timeout 1500 python tools/max_batch.py --model $m --out gpurun_out/maxbatch_$m.json > gpurun_out/maxbatch_$m.log 2>&1
done
