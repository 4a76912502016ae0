mkdir -p gpurun_out/val
o=gpurun_out/val
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/gputest.log 2>&1; tail -3 $o/gputest.log
timeout 600 python __graft_entry__.py --smoke > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 600 python bench.py > $o/bench_default.json 2>$o/bench_default.err; tail -1 $o/bench_default.json | cut -c1-300
timeout 600 python bench.py --model bert-base --micro-batch 8 --stages 4 --micro-batches 16 --steps 5 --cuda-graph > $o/bench_c1_graph.json 2>$o/c1.err; tail -1 $o/bench_c1_graph.json | cut -c1-200
