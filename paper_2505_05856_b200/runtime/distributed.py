"""One process per pipeline stage: the 1F1B scheduler over torch.distributed.

Rank r runs stage x = r+1 of an l = world-size stage plan on its own GPU and
issues exactly `async_ops(l, m, x)` (simulate.py:211-222).  Boundary traffic
is the tensor set of `boundary_bytes` (simulate.py:93-100):

  * forward(j) on stage x>1 first receives stage x-1's boundary activations of
    micro-batch j into its slot buffers, stage x<l sends its own afterwards;
  * backward(j) on stage x<l first receives the gradients of its outgoing
    boundary tensors, stage x>1 sends the gradients of its incoming ones.

Each boundary uses TWO communicators, one per direction.  With one
communicator per stage pair, NCCL serialises a pair's sends and receives on
one stream, and the 1F1B interleaving (send act(j+w) queued before recv
grad(j) on one side, the reverse on the other) can deadlock; with one
communicator per direction each stream carries a single, identically ordered
message sequence (simulate.py's per-direction `_Channel`, :103-114).

Data-parallel replicas of a shallower pipeline (beyond
the reference): with world = l * d ranks, rank r runs stage r % l + 1 of
replica r // l (a replica's stages are consecutive ranks; on NVSwitch the
mapping is free).  Replicas train on different micro-batches with identical
weights: after every backward (1F1B, before the per-micro-batch AdamW) or once
before the iteration's optimizer step (GPipe), each stage all-reduces its flat
fp32 weight gradient over the d ranks holding the same stage (one NCCL
communicator per stage); the 1/d of the mean is folded into the loss-gradient
scale, so every replica applies the same update and the stashed weight
versions stay identical.

The same code runs with the gloo backend on CPU tensors (tests/test_distributed_cpu.py
drives it with a stand-in stage to check ordering, message matching and the
replica gradient sum).
"""

from __future__ import annotations

import os
import time
from typing import Dict, List, Optional, Tuple

import torch
import torch.distributed as dist

from ..planner.balance import SCHEDULE_ASYNC, SCHEDULE_SYNC
from ..planner.schedule import async_ops, sync_ops


class BoundaryChannels:
    """Per-direction process groups for every stage boundary of every replica,
    plus one data-parallel group per stage when there are several replicas.

    fwd[k][p] / bwd[k][p]: boundary p (stage p+1 -> p+2) of replica k;
    dp[p]: the ranks holding stage p+1 in every replica (None if d = 1)."""

    def __init__(self, world: int, stages: Optional[int] = None):
        l = stages or world
        if l < 1 or world % l:
            raise ValueError(f"world size {world} is not a multiple of the stage count {l}")
        self.world, self.stages, self.replicas = world, l, world // l
        self.fwd: List[List[object]] = []
        self.bwd: List[List[object]] = []
        # every rank must create every group, in the same order
        for k in range(self.replicas):
            base = k * l
            fw, bw = [], []
            for p in range(l - 1):
                fw.append(dist.new_group([base + p, base + p + 1]))
                bw.append(dist.new_group([base + p, base + p + 1]))
            self.fwd.append(fw)
            self.bwd.append(bw)
        self.dp: List[Optional[object]] = [None] * l
        if self.replicas > 1:
            self.dp = [dist.new_group([k * l + p for k in range(self.replicas)]) for p in range(l)]

    def position(self, rank: int) -> Tuple[int, int]:
        """(replica k, 0-based stage index p) of a rank."""
        return rank // self.stages, rank % self.stages


def _dp_sync(stage, group) -> None:
    """Sum the stage's weight gradients over its data-parallel group."""
    if group is None:
        return
    for t in stage.dp_grads():
        dist.all_reduce(t, group=group)


def _send(ts: List[torch.Tensor], dst: int, group, copy: bool = False) -> List[object]:
    """isend each tensor; with copy=True the payload is first copied into a
    message buffer on the current stream, so the sender may overwrite its own
    buffer in its next op while the transfer is still in flight."""
    out = []
    for t in ts:
        msg = t.clone() if copy else t.contiguous()
        out.append((dist.isend(msg, dst=dst, group=group), msg))
    return out


def _recv(ts: List[torch.Tensor], src: int, group) -> None:
    works = [dist.irecv(t, src=src, group=group) for t in ts]
    for w in works:
        w.wait()


def run_stage_step(stage, chans: BoundaryChannels, rank: int, world: int, m: int,
                   ids: Optional[torch.Tensor] = None, labels: Optional[torch.Tensor] = None,
                   loss: Optional[torch.Tensor] = None, on_op=None,
                   schedule: str = SCHEDULE_ASYNC) -> None:
    """Run stage rank+1's op list for one iteration of m micro-batches:
    `async_ops` (1F1B) or, for the sync schedule, `sync_ops` (GPipe: all
    forwards, backwards in reverse order, one `optimizer_step` at the end).

    `stage` provides recv_ids/send_ids, recv_buffer/send_buffer(tid, j),
    forward(j, ids, labels, loss_out), backward(j) -> {tid: grad},
    set_recv_grad(tid, t), finish_backward(j), grad_like(tid) (a fresh buffer),
    and, with data-parallel replicas (chans.replicas > 1), dp_grads() -> the
    tensors to all-reduce.  `world` is the stage count of one replica's plan
    times the replica count (chans decides the split)."""
    k, p = chans.position(rank)
    l = chans.stages
    x = p + 1
    fwd_ch, bwd_ch, dp = chans.fwd[k], chans.bwd[k], chans.dp[p]
    pending: List[object] = []
    stream = getattr(stage, "stream", None)
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        ops = sync_ops(l, m, x) if schedule == SCHEDULE_SYNC else async_ops(l, m, x)
        for kind, j, _ in ops:
            if on_op is not None:
                on_op("start", kind, j)
            if kind == "fwd":
                if x > 1:
                    _recv([stage.recv_buffer(t, j) for t in stage.recv_ids], rank - 1,
                          fwd_ch[p - 1])
                stage.forward(j, ids=None if ids is None else ids[j - 1],
                              labels=None if labels is None else labels[j - 1],
                              loss_out=None if loss is None else loss[j - 1:j])
                if x < l:
                    pending += _send([stage.send_buffer(t, j) for t in stage.send_ids], rank + 1,
                                     fwd_ch[p], copy=True)
            else:
                if x < l:
                    bufs = [stage.grad_like(t) for t in stage.send_ids]
                    _recv(bufs, rank + 1, bwd_ch[p])
                    for t, b in zip(stage.send_ids, bufs):
                        stage.set_recv_grad(t, b)
                grads = stage.backward(j)
                if x > 1:
                    pending += _send([grads[t] for t in stage.recv_ids], rank - 1, bwd_ch[p - 1])
                if schedule != SCHEDULE_SYNC:
                    _dp_sync(stage, dp)  # before this micro-batch's AdamW
                stage.finish_backward(j)
            if on_op is not None:
                on_op("end", kind, j)
        if schedule == SCHEDULE_SYNC:
            _dp_sync(stage, dp)
            stage.optimizer_step()
        for w, _ in pending:
            w.wait()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def init_process_group_from_env(backend: str) -> Tuple[int, int]:
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size()


def run_bench_distributed(args) -> None:
    """bench.py at N>1 (torchrun): an l-stage plan (l = --stages, default N), one
    stage per GPU; N/l data-parallel replicas of it when l < N."""
    import json
    from .. import kernels as K
    from .. import planner as P
    from .._lib import init_device
    from .graph import profile_graph
    from .model import PRESETS, build_nodes, init_params, synthetic_batch
    from .stage import StageExecutor

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    init_device(local)
    rank, world = init_process_group_from_env("nccl")
    stages = args.stages or world
    chans = BoundaryChannels(world, stages)
    rep_k, pos = chans.position(rank)
    d = chans.replicas
    cfg = PRESETS[args.model]
    b, m = args.micro_batch, args.micro_batches
    g = profile_graph(cfg, b)
    plan = P.plan(g, P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC,
                                  capacity=int(args.capacity_gib * (1 << 30)), bandwidth=64 << 30))
    lo, hi = P.stage_bounds(plan.cuts, len(g))[pos]
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    stage = StageExecutor(cfg=cfg, g=g, nodes=build_nodes(cfg), lo=lo, hi=hi, stage=pos + 1,
                          stages=stages, micro_batch=b, memopt=plan.memopt[pos],
                          init=init_params(cfg, 0), device=dev, stream=stream, dp_replicas=d)
    ids, labels = synthetic_batch(cfg, m, b, seed=rep_k)  # each replica its own data
    ids_d = ids.to(dev) if stage.needs_ids else None
    lab_d = labels.to(dev) if stage.is_last else None
    loss = torch.zeros(m, device=dev) if stage.is_last else None
    torch.cuda.synchronize()

    def step():
        run_stage_step(stage, chans, rank, world, m, ids_d, lab_d, loss)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = K.INSTR.launches
    clocks = None
    if rank == 0:
        try:
            import sys
            sys.path.insert(0, os.getcwd())
            from bench import Clocks
            clocks = Clocks(local)
            clocks.start()
        except Exception:  # clock sampling is evidence, not part of the run
            clocks = None
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks is not None else None
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    launches = torch.tensor([(K.INSTR.launches - l0) // args.steps], device=dev, dtype=torch.int64)
    dist.all_reduce(launches)
    value = args.steps * m * b * d / (ms.item() / 1e3)

    # e2e: inputs copied H2D from pinned memory on the ranks that embed, the loss
    # vector read back on the last rank, every step; wall time, max over ranks
    ids_h = ids.pin_memory() if stage.needs_ids else None
    lab_h = labels.pin_memory() if stage.is_last else None
    loss_h = torch.empty(m, dtype=torch.float32).pin_memory() if stage.is_last else None
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            if ids_h is not None:
                ids_d.copy_(ids_h, non_blocking=True)
            if lab_h is not None:
                lab_d.copy_(lab_h, non_blocking=True)
        run_stage_step(stage, chans, rank, world, m, ids_d, lab_d, loss)
        if loss_h is not None:
            with torch.cuda.stream(stream):
                loss_h.copy_(loss, non_blocking=True)
        stream.synchronize()
    wall = torch.tensor([time.perf_counter() - t0], device=dev)
    dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    h2d = torch.tensor([(ids.numel() * ids.element_size() if stage.needs_ids else 0)
                        + (labels.numel() * labels.element_size() if stage.is_last else 0)],
                       device=dev, dtype=torch.int64)
    dist.all_reduce(h2d)
    e2e = {"value": args.steps * m * b * d / wall.item(), "unit": "samples/s",
           "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": m * 4 * d}
    if rank == 0:
        out = {"metric": "samples/sec at 1/2/4/8 stages; max trainable batch under per-GPU mem cap",
               "value": round(value, 2), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms.item() / args.steps, 3),
               "higher_is_better": True, "scaling": "strong" if d == 1 else "weak",
               "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic",
               "config": {"workload": f"{args.model} s{cfg.seq}, {stages}-stage DawnPiper 1F1B plan, "
                                      f"one stage per GPU, NCCL P2P boundaries, b={b}, m={m}"
                                      + (f", {d} data-parallel replicas (per-update gradient "
                                         f"all-reduce)" if d > 1 else ""),
                          "model": args.model, "global_batch": b * m * d, "seq_len": cfg.seq,
                          "micro_batch": b, "micro_batches": m, "stages": stages, "replicas": d,
                          "cuts": list(plan.cuts.positions),
                          "parallelism": f"pp{stages}" + (f"xdp{d}" if d > 1 else "")},
               "gpu_launches": int(launches.item()), "e2e": e2e, "clocks": clk,
               "roofline": None, "model_tflops": round(value * cfg.flops_per_sample() / 1e12, 1)}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
