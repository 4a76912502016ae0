#!/bin/bash
# the one-process-per-stage path (NCCL send/recv, run_bench_distributed) with
# two ranks sharing the single GPU of a gpurun box (DPN_SINGLE_DEVICE test hook)
set -x
mkdir -p gpurun_out
export NCCL_DEBUG=WARN
DPN_SINGLE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --micro-batch 4 --micro-batches 8 > gpurun_out/bench_dist2.json 2> gpurun_out/bench_dist2.err
echo "rc=$?" >> gpurun_out/bench_dist2.err
timeout 300 python tools/swap_bw.py > gpurun_out/swap_bw.txt 2>&1
