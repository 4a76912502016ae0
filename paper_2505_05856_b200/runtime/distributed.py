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

import json
import os
import time
from pathlib import Path
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


class _Sent:
    """An in-flight send; `wait` orders the caller's stream after it (once:
    gloo's send work consumes one completion per wait)."""

    def __init__(self, work, payload):
        self.work, self.payload = work, payload

    def wait(self):
        if self.work is not None:
            self.work.wait()
            self.work = self.payload = None


class _Inbound:
    """A posted receive; `wait` returns the landed tensor on the caller's device."""

    def __init__(self, work, landing, target=None):
        self.work, self.landing, self.target = work, landing, target

    def wait(self) -> torch.Tensor:
        self.work.wait()
        if self.target is not None:  # host-staged: copy into the device buffer
            self.target.copy_(self.landing, non_blocking=True)
            return self.target
        return self.landing


class Wire:
    """How boundary tensors travel over a process group.

    NCCL moves device tensors directly (P2P over NVLink / NVSwitch between
    the stages' GPUs; PG-NCCL records the tensors on its stream, so a buffer
    the sender drops is not recycled before the transfer has read it).  Gloo
    only moves host tensors: device tensors are staged through host copies
    (the CPU tests, and several stage processes sharing one GPU -- NCCL
    refuses two ranks on one device)."""

    def __init__(self, backend: Optional[str] = None):
        self.nccl = (backend or dist.get_backend()) == "nccl"

    def send(self, t: torch.Tensor, dst: int, group) -> _Sent:
        if self.nccl:
            t = t.contiguous()
        else:  # gloo reads the buffer asynchronously: hand it a private host copy
            t = t.detach().to("cpu", copy=True)
        return _Sent(dist.isend(t, dst=dst, group=group), t)

    def recv(self, like: torch.Tensor, src: int, group) -> _Inbound:
        if self.nccl or like.device.type == "cpu":
            return _Inbound(dist.irecv(like, src=src, group=group), like)
        landing = torch.empty(like.shape, dtype=like.dtype)
        return _Inbound(dist.irecv(landing, src=src, group=group), landing, like)


def run_stage_step(stage, chans: BoundaryChannels, rank: int, world: int, m: int,
                   ids: Optional[torch.Tensor] = None, labels: Optional[torch.Tensor] = None,
                   loss: Optional[torch.Tensor] = None, on_op=None,
                   schedule: str = SCHEDULE_ASYNC, wire: Optional[Wire] = None) -> None:
    """Run stage rank+1's op list for one iteration of m micro-batches:
    `async_ops` (1F1B) or, for the sync schedule, `sync_ops` (GPipe: all
    forwards, backwards in reverse order, one `optimizer_step` at the end).

    `stage` provides recv_ids/send_ids, recv_buffer/send_buffer(tid, j),
    forward(j, ids, labels, loss_out), backward(j) -> {tid: grad},
    set_recv_grad(tid, t), finish_backward(j), grad_like(tid) (a fresh buffer),
    and, with data-parallel replicas (chans.replicas > 1), dp_grads() -> the
    tensors to all-reduce.  `world` is the stage count of one replica's plan
    times the replica count (chans decides the split).

    A stage that also provides recv_like(tid) / adopt_recv(tid, j, t) /
    release_send_buffer(tid, j) (the B200 StageExecutor) gets the overlapped
    protocol: the receive of the next forward's activations and of the next
    backward's gradients is posted as soon as the current op is issued, into
    fresh buffers the stage adopts (no copy), so transfers overlap compute;
    boundary activations are sent from the stage's own buffers (released to
    the transfer when its backward does not read them) without a copy, and a
    slot's buffers are rewritten only after its last send has completed."""
    k, p = chans.position(rank)
    l = chans.stages
    x = p + 1
    fwd_ch, bwd_ch, dp = chans.fwd[k], chans.bwd[k], chans.dp[p]
    wire = wire or Wire()
    overlapped = all(hasattr(stage, a) for a in ("recv_like", "adopt_recv", "release_send_buffer"))
    pending: List[_Sent] = []
    slot_sends: Dict[int, List[_Sent]] = {}
    acts_in: Dict[int, List[_Inbound]] = {}
    grads_in: Dict[int, List[_Inbound]] = {}
    stream = getattr(stage, "stream", None)
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()

    def post_acts(j: int) -> None:
        if x > 1 and j not in acts_in:
            acts_in[j] = [wire.recv(stage.recv_like(t), rank - 1, fwd_ch[p - 1])
                          for t in stage.recv_ids]

    def post_grads(j: int) -> None:
        if x < l and j not in grads_in:
            grads_in[j] = [wire.recv(stage.grad_like(t), rank + 1, bwd_ch[p])
                           for t in stage.send_ids]

    with ctx:
        if loss is not None:
            loss.zero_()  # the head accumulates each micro-batch's loss into its entry
        ops = sync_ops(l, m, x) if schedule == SCHEDULE_SYNC else async_ops(l, m, x)
        nxt_f = [j for kd, j, _ in ops if kd == "fwd"]
        nxt_b = [j for kd, j, _ in ops if kd == "bwd"]
        for kind, j, _ in ops:
            if on_op is not None:
                on_op("start", kind, j)
            if kind == "fwd":
                nxt_f.pop(0)
                if overlapped:
                    slot = getattr(stage, "slot_of", lambda mb: mb)(j)
                    for s in slot_sends.pop(slot, []):
                        s.wait()  # the slot's buffers are about to be rewritten
                    if x > 1:
                        post_acts(j)
                        for t, h in zip(stage.recv_ids, acts_in.pop(j)):
                            stage.adopt_recv(t, j, h.wait())
                elif x > 1:
                    hs = [wire.recv(stage.recv_buffer(t, j), rank - 1, fwd_ch[p - 1])
                          for t in stage.recv_ids]
                    for h in hs:
                        h.wait()
                stage.forward(j, ids=None if ids is None else ids[j - 1],
                              labels=None if labels is None else labels[j - 1],
                              loss_out=None if loss is None else loss[j - 1:j])
                if x < l:
                    sent = []
                    for t in stage.send_ids:
                        msg = stage.release_send_buffer(t, j) if overlapped else None
                        sent.append(wire.send(msg if msg is not None else stage.send_buffer(t, j),
                                              rank + 1, fwd_ch[p]))
                    pending += sent
                    if overlapped:
                        slot_sends[slot] = sent
            else:
                nxt_b.pop(0)
                if x < l:
                    if overlapped:
                        post_grads(j)
                        hs = grads_in.pop(j)
                    else:
                        hs = [wire.recv(stage.grad_like(t), rank + 1, bwd_ch[p])
                              for t in stage.send_ids]
                    for t, h in zip(stage.send_ids, hs):
                        stage.set_recv_grad(t, h.wait())
                grads = stage.backward(j)
                if x > 1:
                    pending += [wire.send(grads[t], rank - 1, bwd_ch[p - 1]) for t in stage.recv_ids]
                if schedule != SCHEDULE_SYNC:
                    _dp_sync(stage, dp)  # before this micro-batch's AdamW
                stage.finish_backward(j)
            if overlapped:  # receives of the next forward / backward, posted early
                if nxt_f:
                    post_acts(nxt_f[0])
                if nxt_b:
                    post_grads(nxt_b[0])
            if on_op is not None:
                on_op("end", kind, j)
        if schedule == SCHEDULE_SYNC:
            _dp_sync(stage, dp)
            stage.optimizer_step()
        for w in pending:
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
    # the planner is fed measured B200 per-node times: rank 0 profiles the
    # whole model on its GPU and every rank plans from the same numbers
    t_prof = time.perf_counter()
    times = [None]
    if rank == 0:
        from .profiler import measure_node_times
        times[0] = measure_node_times(cfg, b, device=local, iters=args.profile_iters, warmup=3)
        torch.cuda.empty_cache()
    dist.broadcast_object_list(times, src=0)
    t_prof = time.perf_counter() - t_prof
    g = profile_graph(cfg, b, times=times[0], name=f"{cfg.name}_b{b}")
    t_plan = time.perf_counter()
    plan = P.plan(g, P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC,
                                  capacity=int(args.capacity_gib * (1 << 30)), bandwidth=64 << 30))
    t_plan = time.perf_counter() - t_plan
    lo, hi = P.stage_bounds(plan.cuts, len(g))[pos]
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    stage = StageExecutor(cfg=cfg, g=g, nodes=build_nodes(cfg), lo=lo, hi=hi, stage=pos + 1,
                          stages=stages, micro_batch=b, memopt=plan.memopt[pos],
                          init=init_params(cfg, 0), device=dev, stream=stream, dp_replicas=d)
    from .pipeline import RunConfig
    knobs = RunConfig(micro_batches=m, micro_batch_size=b)
    stage.d2h_budget, stage.prefetch_budget = knobs.d2h_budget, knobs.swap_prefetch
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
    # roofline of the dominant kernel: every GEMM launch of one step on every
    # rank, CUDA events on the rank's stream; summed FLOPs / summed time
    K.INSTR.gemm_events = []
    run_stage_step(stage, chans, rank, world, m, ids_d, lab_d, loss)
    torch.cuda.synchronize()
    evs = K.INSTR.gemm_events
    K.INSTR.gemm_events = None
    fl_ms = torch.tensor([float(sum(e[0] for e in evs)), sum(e[1].elapsed_time(e[2]) for e in evs),
                          float(len(evs))], device=dev, dtype=torch.float64)
    dist.all_reduce(fl_ms)
    peaks_f = Path(os.getcwd()) / "MEASURED_PEAKS.json"
    peaks = json.loads(peaks_f.read_text()) if peaks_f.exists() else {}
    peak = peaks.get("bf16_tflops_sustained", 1400.0)
    achieved = fl_ms[0].item() / (fl_ms[1].item() / 1e3) / 1e12 if fl_ms[1].item() > 0 else 0.0
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": "dpn gemm_kernel (tcgen05), all launches of one step on all ranks",
                "launches_per_step": int(fl_ms[2].item()),
                "gemm_ms_per_step_summed_over_ranks": round(fl_ms[1].item(), 3),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else "fallback"}
    cpu = None
    if rank == 0 and not getattr(args, "no_cpu_baseline", False):
        try:
            import sys
            sys.path.insert(0, os.getcwd())
            from bench import CpuPort
            port = CpuPort(args.model, plan.cuts.positions)
            port.step()
            dt = port.step()
            cpu = {"value": round(port.samples / dt, 4), "unit": "samples/s", "cores": port.cores,
                   "kind": "port", "sample": port.sample + f", {dt:.1f} s"}
        except Exception as e:  # the CPU baseline is a reported reference, not the run
            cpu = {"error": str(e)[:200]}
    dist.barrier()
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
               "roofline": roofline, "model_tflops": round(value * cfg.flops_per_sample() / 1e12, 1),
               "cpu_baseline": cpu,
               "profile": f"measured B200 node times on rank 0 ({args.profile_iters} iters, "
                          f"{t_prof:.1f} s, broadcast); plan {t_plan:.2f} s"}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
