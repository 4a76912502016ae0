#!/bin/bash
# Round-2 end-of-session evidence on one B200: GPU tests, smoke, bench lines.
mkdir -p gpurun_out/final_s3
o=gpurun_out/final_s3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/gputest.log 2>&1; tail -3 $o/gputest.log
timeout 600 python __graft_entry__.py --smoke > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 600 python bench.py > $o/bench_default.json 2>$o/bench_default.err; tail -1 $o/bench_default.json | cut -c1-200
for l in 1 2 4; do
  timeout 600 python bench.py --stages $l --steps 3 --no-cpu-baseline > $o/bench_stages$l.json 2>/dev/null; tail -1 $o/bench_stages$l.json | cut -c1-160
done
timeout 600 python bench.py --model bert-base --micro-batch 8 --stages 4 --micro-batches 16 --steps 5 > $o/bench_c1.json 2>/dev/null; tail -1 $o/bench_c1.json | cut -c1-160
timeout 600 python bench.py --model bert-base --micro-batch 8 --stages 4 --micro-batches 16 --steps 5 --cuda-graph --no-cpu-baseline > $o/bench_c1_graph.json 2>/dev/null; tail -1 $o/bench_c1_graph.json | cut -c1-160
timeout 600 python bench.py --model gpt2-xl --micro-batch 4 --steps 3 --no-cpu-baseline > $o/bench_gpt2xl.json 2>/dev/null; tail -1 $o/bench_gpt2xl.json | cut -c1-160
timeout 600 python bench.py --model t5-large --micro-batch 16 --steps 3 --no-cpu-baseline > $o/bench_t5.json 2>/dev/null; tail -1 $o/bench_t5.json | cut -c1-160
timeout 600 python bench.py --model amoebanet-d --micro-batch 64 --steps 3 --no-cpu-baseline > $o/bench_amoeba.json 2>/dev/null; tail -1 $o/bench_amoeba.json | cut -c1-160
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_reference.json 2>/dev/null; tail -1 $o/bench_reference.json | cut -c1-160
