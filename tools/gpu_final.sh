#!/bin/bash
# Full GPU suite, smoke, default bench, max-batch re-measurement (one B200).
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
[ -n "$NO_MAXBATCH" ] && exit 0
timeout 900 python tools/max_batch.py --model amoebanet-d --b-max 1024 --out gpurun_out/maxbatch_amoebanet-d.json > gpurun_out/maxbatch_amoebanet-d.log 2>&1
timeout 900 python tools/max_batch.py --model t5-large --b-max 128 --host-cap-gib 64 --out gpurun_out/maxbatch_t5-large.json > gpurun_out/maxbatch_t5-large.log 2>&1
timeout 900 python tools/max_batch.py --model gpt2-xl --b-max 64 --host-cap-gib 64 --out gpurun_out/maxbatch_gpt2-xl.json > gpurun_out/maxbatch_gpt2-xl.log 2>&1
