"""The B200 pipeline run: `run(plan, g, cfg) -> RunReport`.

This replaces the reference's analytic `simulate(plan, g, cfg)`
(simulate.py:130-166) with a real 1F1B training run of the plan's partition:

  * one `StageExecutor` per plan stage (`stage_bounds(plan.cuts)`), executing
    that stage's memopt actions for real;
  * every stage issues exactly `async_ops(l, m, x)` (simulate.py:211-222):
    min(l-x, m) warm-up forwards, (F, B) pairs, then the drain;
  * boundary activations / gradients are the tensors of `boundary_bytes`
    (simulate.py:93-100), moved per micro-batch: device-to-device when stages
    share a GPU, cudaMemcpyPeerAsync when they are on peer GPUs of one
    process, NCCL send/recv (torch.distributed) when each stage is its own
    process (`run_distributed`).

With all stages on one GPU (`devices=[0]`, the 1-GPU bench case) a single
host thread issues the stages' op lists interleaved by the same readiness
walk the reference simulator uses (simulate.py:244-282); dependencies are
then satisfied by stream order.

The report is a superset of SimReport: the same fields, measured from CUDA
events, plus per-micro-batch losses, samples/s and the memory actually held.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from .. import kernels as K
from .._lib import init_device
from ..planner.balance import SCHEDULE_ASYNC, SCHEDULE_SYNC
from ..planner.profile import ComputationGraph
from ..planner.schedule import SimEvent, async_iteration, async_ops, inflight_depth
from ..planner.search import PartitionPlan, stage_bounds
from .model import AdamWConfig, TransformerConfig, build_nodes, init_params
from .stage import StageExecutor


@dataclass(frozen=True)
class RunConfig:
    micro_batches: int
    micro_batch_size: int
    devices: Tuple[int, ...] = (0,)
    seed: int = 0
    opt: AdamWConfig = AdamWConfig()
    trace: bool = True
    capacity: Optional[int] = None  # per-GPU byte cap enforced on the caching allocator
    # co-located stages on one GPU run on their own CUDA streams (cross-stage
    # dependencies through events), so independent work of different stages
    # -- what separate GPUs would run in parallel -- can overlap on the device
    concurrent_stages: bool = True
    # `run` only: after the timed steps, run every stage alone on its GPU with
    # its real op list (runtime/memprobe.py) and report those measured device
    # peaks as per_stage_peak (otherwise: the stage's static buffer bytes)
    measure_stage_peaks: bool = False
    # swap engine knobs for throughput runs (StageExecutor defaults hold
    # memory to the planner's model: 256 MiB of D2H in flight, no early
    # prefetch): offloads may queue up to d2h_budget bytes behind the forward
    # and the next micro-batch's swap-ins start at the end of a backward, up
    # to swap_prefetch bytes -- both held that much longer than the model
    # assumes (tools/memopt_knobs.py: GPT-2 XL stage 1, b=16, 40 GiB cap:
    # 80 -> 44 ms per micro-batch, peak +1.3 GB)
    d2h_budget: int = 1 << 30
    swap_prefetch: int = 2 << 30
    # one device arena per stage (runtime/arena.py) of `capacity` bytes: the
    # stage's own cap (as on its own GPU) and its measured peak; the arenas
    # are reserved up front, so the stages sharing a device must fit it
    arenas: bool = False
    # replay each iteration as one captured CUDA graph (co-located async
    # plans without memopt actions): the host issues one graph launch per step
    # instead of every kernel -- what a small-b / small-model step needs when
    # ~20k ctypes launches take longer than the GPU work (C1: 64 ms of host
    # issue for 64 ms of GPU time, tools/host_profile.py)
    cuda_graph: bool = False

    def __post_init__(self):
        if self.micro_batches < 1:
            raise ValueError("need at least one micro-batch")
        if self.micro_batch_size < 1:
            raise ValueError("micro-batch size must be positive")


@dataclass(frozen=True)
class RunReport:
    # SimReport fields (simulate.py:60-79), measured
    per_stage_peak: Tuple[int, ...]
    iteration_time: float
    bubble_ratio: float
    waste_ratio: float
    trace: Tuple[SimEvent, ...]
    makespan: int
    capacity_exceeded: Tuple[int, ...]
    # run-only fields
    losses: Tuple[float, ...] = ()
    samples_per_s: float = 0.0
    step_time_us: float = 0.0
    device_peak_bytes: int = 0
    per_stage_peak_source: str = "static"

    def to_doc(self) -> dict:
        return {
            "per_stage_peak_bytes": list(self.per_stage_peak),
            "iteration_time_us": self.iteration_time,
            "bubble_ratio": self.bubble_ratio,
            "waste_ratio": self.waste_ratio,
            "makespan_us": self.makespan,
            "capacity_exceeded_stages": list(self.capacity_exceeded),
            "events": len(self.trace),
            "losses": list(self.losses),
            "samples_per_s": self.samples_per_s,
            "step_time_us": self.step_time_us,
            "device_peak_bytes": self.device_peak_bytes,
            "per_stage_peak_source": self.per_stage_peak_source,
        }


def sync_order(stages: int, m: int) -> List[Tuple[int, str, int]]:
    """GPipe issue order of simulate.py:169-208: every forward (micro-batch j
    through stages 1..l), then every backward in reverse micro-batch order
    (j = m..1 through stages l..1).  Per stage this is `sync_ops`."""
    out = [(x, "fwd", j) for j in range(1, m + 1) for x in range(1, stages + 1)]
    out += [(x, "bwd", j) for j in range(m, 0, -1) for x in range(stages, 0, -1)]
    return out


def colocated_order(stages: int, m: int) -> List[Tuple[int, str, int]]:
    """Interleave the stages' 1F1B op lists by dependency readiness, scanning
    stages in order exactly like simulate.py:244-282 (without durations).
    Returns (stage 1-based, kind, micro-batch)."""
    ops = [async_ops(stages, m, x + 1) for x in range(stages)]
    ptr = [0] * stages
    fwd_done = [set() for _ in range(stages)]
    bwd_done = [set() for _ in range(stages)]
    out = []
    left = sum(len(o) for o in ops)
    while left:
        moved = False
        for x in range(stages):
            while ptr[x] < len(ops[x]):
                kind, j, _ = ops[x][ptr[x]]
                if kind == "fwd":
                    ok = x == 0 or j in fwd_done[x - 1]
                else:
                    ok = (j in fwd_done[x]) if x == stages - 1 else (j in bwd_done[x + 1])
                if not ok:
                    break
                out.append((x + 1, kind, j))
                (fwd_done if kind == "fwd" else bwd_done)[x].add(j)
                ptr[x] += 1
                left -= 1
                moved = True
        if not moved:
            raise RuntimeError("schedule deadlock; op lists are inconsistent")
    return out


class Pipeline:
    """All stages of a plan in one process (one or several local GPUs)."""

    def __init__(self, model: TransformerConfig, g: ComputationGraph, plan: PartitionPlan,
                 cfg: RunConfig):
        if plan.schedule not in (SCHEDULE_ASYNC, SCHEDULE_SYNC):
            raise ValueError(f"unknown schedule {plan.schedule!r}")
        self.sync = plan.schedule == SCHEDULE_SYNC
        bounds = stage_bounds(plan.cuts, len(g))
        if len(g) != len(build_nodes(model)):
            raise ValueError("graph does not describe this model (node count mismatch)")
        self.model, self.g, self.plan, self.cfg = model, g, plan, cfg
        self.l = len(bounds)
        self.m = cfg.micro_batches
        devs = list(cfg.devices)
        self.stage_dev = [devs[min(x * len(devs) // self.l, len(devs) - 1)] for x in range(self.l)]
        for d in set(self.stage_dev):
            init_device(d)
        for a in set(self.stage_dev):
            for b in set(self.stage_dev):
                if a != b:
                    from .._lib import check, lib
                    check(lib().dpn_enable_peer(a, b), "dpn_enable_peer")
        self.arenas = None
        if cfg.arenas:
            if cfg.capacity is None:
                raise ValueError("per-stage arenas need a capacity")
            from .arena import StageArena
            self.arenas = [StageArena(d, cfg.capacity) for d in self.stage_dev]
        elif cfg.capacity is not None:
            # the plan's capacity is per stage; stages sharing a GPU share its cap
            for d in set(self.stage_dev):
                total = torch.cuda.get_device_properties(d).total_memory
                share = cfg.capacity * self.stage_dev.count(d)
                torch.cuda.set_per_process_memory_fraction(min(1.0, share / total), d)
        self.streams = {d: torch.cuda.Stream(device=d) for d in set(self.stage_dev)}
        # one stream per stage when several stages share a device (see RunConfig)
        self.multi = cfg.concurrent_stages and len(set(self.stage_dev)) < self.l
        self.stage_streams = [torch.cuda.Stream(device=d) if self.multi else self.streams[d]
                              for d in self.stage_dev]
        # True: concurrent stages are chained op by op (issue order), e.g. to
        # time kernels in isolation
        self.serialize = False
        nodes = build_nodes(model)
        init = init_params(model, cfg.seed)
        self.stages: List[StageExecutor] = []
        for x, (lo, hi) in enumerate(bounds, start=1):
            d = self.stage_dev[x - 1]
            with torch.cuda.device(d), self._arena(x - 1):
                self.stages.append(StageExecutor(
                    cfg=model, g=g, nodes=nodes, lo=lo, hi=hi, stage=x, stages=self.l,
                    micro_batch=cfg.micro_batch_size, memopt=plan.memopt[x - 1], init=init,
                    device=torch.device("cuda", d), stream=self.stage_streams[x - 1], opt=cfg.opt,
                    schedule=plan.schedule, micro_batches=self.m))
                self.stages[-1].d2h_budget = cfg.d2h_budget
                self.stages[-1].prefetch_budget = cfg.swap_prefetch
        self.order = sync_order(self.l, self.m) if self.sync else colocated_order(self.l, self.m)
        self._graph = None
        first_dev = self.stage_dev[0]
        self.loss = torch.zeros(self.m, dtype=torch.float32, device=torch.device("cuda", self.stage_dev[-1]))
        self.static_bytes = [self._stage_bytes(s) for s in self.stages]
        for d in set(self.stage_dev):
            torch.cuda.synchronize(d)  # parameter init (default stream) before the run streams

    def _arena(self, x: int):
        """Allocation context of stage index x (0-based)."""
        if self.arenas is None:
            import contextlib
            return contextlib.nullcontext()
        return self.arenas[x].active()

    def arena_peaks(self) -> Optional[List[int]]:
        return None if self.arenas is None else [a.stats()[1] for a in self.arenas]

    @staticmethod
    def _stage_bytes(s: StageExecutor) -> int:
        tot = 0
        for t in (s.params.master, s.params.m, s.params.v, s.params.grad, s.params.ring):
            tot += t.numel() * t.element_size()
        for d in s.slot_buf:
            tot += sum(t.numel() * t.element_size() for t in d.values())
        return tot

    def _peer_msg(self, src: torch.Tensor, d_src: int, d_dst: int, sst, dst_st) -> torch.Tensor:
        """Copy src (on device d_src, live in stream sst) into a fresh buffer on
        d_dst, pushed by the sender: the buffer is allocated in the receiver's
        stream order, the copy runs on sst (so the sender cannot overwrite or
        free src before it is read), and the receiver waits on the returned
        buffer through the caller's event."""
        with torch.cuda.device(d_dst), torch.cuda.stream(dst_st):
            msg = torch.empty(src.shape, dtype=src.dtype, device=torch.device("cuda", d_dst))
            ready = torch.cuda.Event()
            ready.record(dst_st)
        sst.wait_event(ready)
        K.copy_d2d(msg, src, dst_dev=d_dst, src_dev=d_src, stream=sst)
        msg.record_stream(sst)
        return msg

    def _send_fwd_streams(self, x: int, j: int):
        """Concurrent co-located stages: the sender copies its boundary
        activations into message buffers on its own stream; the receiver's
        stream waits on the recorded event before delivering."""
        src = self.stages[x - 1]
        sst, dst_st = self.stage_streams[x - 1], self.stage_streams[x]
        d_src, d_dst = self.stage_dev[x - 1], self.stage_dev[x]
        out = {}
        with torch.cuda.stream(sst):
            for tid in src.send_ids:
                if d_src != d_dst:  # stages on different GPUs: peer copy
                    out[tid] = self._peer_msg(src.send_buffer(tid, j), d_src, d_dst, sst, dst_st)
                    continue
                # buffers the sender's backward never reads change owner (no copy)
                msg = src.release_send_buffer(tid, j)
                if msg is None:
                    a = src.send_buffer(tid, j)
                    msg = torch.empty_like(a)
                    K.copy_d2d(msg, a, dst_dev=d_src, src_dev=d_src, stream=sst)
                msg.record_stream(dst_st)
                out[tid] = msg
            ev = torch.cuda.Event()
            ev.record(sst)
        return out, ev

    def _send_bwd_streams(self, x: int, grads: Dict[str, torch.Tensor]):
        """Gradients of stage x's inputs handed to stage x-1."""
        sst, dst = self.stage_streams[x - 1], self.stage_streams[x - 2]
        d_src, d_dst = self.stage_dev[x - 1], self.stage_dev[x - 2]
        out = {}
        seen = set()
        with torch.cuda.stream(sst):
            for tid, g in grads.items():
                if d_src != d_dst:
                    out[tid] = self._peer_msg(g, d_src, d_dst, sst, dst)
                    continue
                # the sender drops its gradient buffers after this backward, so they
                # are handed over as they are; one buffer aliased by two tensors'
                # gradients is copied (the receiver may update either in place)
                if g.data_ptr() in seen:
                    g = g.clone()
                seen.add(g.data_ptr())
                g.record_stream(dst)
                out[tid] = g
            ev = torch.cuda.Event()
            ev.record(sst)
        return out, ev

    def _send_fwd(self, x: int, j: int) -> Dict[str, torch.Tensor]:
        """Stage x (1-based) sends micro-batch j's boundary activations: they are
        copied into message buffers owned by the receiver (the sender's own
        buffers are reused by its next forward, and the receiver may not have
        a free slot yet -- exactly like a posted NCCL send)."""
        src = self.stages[x - 1]
        d_src, d_dst = self.stage_dev[x - 1], self.stage_dev[x]
        sst, st = self.streams[d_src], self.streams[d_dst]
        out = {}
        for tid in src.send_ids:
            a = src.send_buffer(tid, j)
            if d_src != d_dst:
                out[tid] = self._peer_msg(a, d_src, d_dst, sst, st)
            else:
                with torch.cuda.stream(st):
                    msg = torch.empty_like(a)
                    K.copy_d2d(msg, a, dst_dev=d_dst, src_dev=d_src, stream=st)
                out[tid] = msg
        if d_src != d_dst:
            ev = torch.cuda.Event()
            ev.record(sst)
            st.wait_event(ev)
        return out

    def _deliver_fwd(self, x: int, j: int, msgs: Dict[str, torch.Tensor]) -> None:
        """Receiver side: land the messages in stage x's slot for micro-batch j."""
        dst = self.stages[x - 1]
        st = self.streams[self.stage_dev[x - 1]]
        for tid, msg in msgs.items():
            K.copy_d2d(dst.recv_buffer(tid, j), msg, dst_dev=self.stage_dev[x - 1],
                       src_dev=self.stage_dev[x - 1], stream=st)

    def _send_bwd(self, x: int, grads: Dict[str, torch.Tensor]) -> Dict[str, torch.Tensor]:
        # x is the sending stage (1-based); returns fresh buffers owned by stage x-1
        d_src, d_dst = self.stage_dev[x - 1], self.stage_dev[x - 2]
        sst, st = self.streams[d_src], self.streams[d_dst]
        out = {}
        for tid, gsrc in grads.items():
            if d_src != d_dst:
                out[tid] = self._peer_msg(gsrc, d_src, d_dst, sst, st)
            else:
                with torch.cuda.stream(st):
                    gdst = torch.empty_like(gsrc)
                    K.copy_d2d(gdst, gsrc, dst_dev=d_dst, src_dev=d_src, stream=st)
                out[tid] = gdst
        if d_src != d_dst:
            ev = torch.cuda.Event()
            ev.record(sst)
            st.wait_event(ev)
        return out

    def step(self, ids: torch.Tensor, labels: torch.Tensor, events: Optional[list] = None) -> torch.Tensor:
        """One training iteration (m micro-batches).  ids/labels: int32 [m, b*s] on
        the first / last stage's device.  Returns the device loss vector [m]."""
        if self.cfg.cuda_graph and events is None and not self.serialize:
            return self._graph_step(ids, labels)
        loss = self._eager_step(ids, labels, events)
        if self._graph is not None:  # keep the replay invariant: newest weights in the start slot
            self._restore_ring()
        return loss

    def _restore_ring(self) -> None:
        dev = self.stage_dev[0]
        main = self.streams[dev]
        for s, l0 in zip(self.stages, self._graph_start):
            if s.params.latest != l0:
                K.copy_d2d(s.params.ring[l0], s.params.ring[s.params.latest], dst_dev=dev,
                           src_dev=dev, stream=main)
                s.params.latest = l0

    # ---- CUDA-graph mode --------------------------------------------------------

    def _graph_step(self, ids: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        dev = self.stage_dev[0]
        main = self.streams[dev]
        if self._graph is None:
            self._capture(ids, labels)
        caller = torch.cuda.current_stream(dev)
        ready = torch.cuda.Event()
        ready.record(caller)
        main.wait_event(ready)
        with torch.cuda.stream(main):
            self._gids.copy_(ids, non_blocking=True)
            self._glabels.copy_(labels, non_blocking=True)
            self._graph.replay()
        done = torch.cuda.Event()
        done.record(main)
        caller.wait_event(done)
        return self.loss

    def _capture(self, ids: torch.Tensor, labels: torch.Tensor) -> None:
        """Warm up eagerly on static input buffers, then capture one iteration.

        A captured iteration replays with the addresses it was recorded with,
        so (1) every tensor the stages hold when capture starts is kept alive
        (buffers handed over during the step are replaced by graph-pool ones),
        (2) each stage's newest weights are copied back into the ring slot they
        occupied at capture start, so every replay starts from the same ring
        state, and (3) AdamW reads its step count from device memory."""
        if len(self.streams) != 1 or self.sync:
            raise ValueError("CUDA-graph mode runs co-located async (1F1B) plans")
        if any(m.actions for m in self.plan.memopt):
            raise ValueError("CUDA-graph mode runs plans without swap / recompute actions")
        dev = self.stage_dev[0]
        main = self.streams[dev]
        for s in self.stages:
            s.params.device_step = True
            s.params.step_dev.fill_(s.params.step)
        self._gids = ids.clone()
        self._glabels = labels.clone()
        # the warm-up iterations must not train: snapshot and restore the state
        saved = [(s.params.latest, s.params.step,
                  [t.clone() for t in (s.params.master, s.params.m, s.params.v, s.params.ring,
                                       s.params.step_dev)]) for s in self.stages]
        for _ in range(2):  # lazy allocations, workspaces, kernel attributes
            self._eager_step(self._gids, self._glabels, None)
        torch.cuda.synchronize(dev)
        for s, (latest, step, ts) in zip(self.stages, saved):
            for dst, src in zip((s.params.master, s.params.m, s.params.v, s.params.ring,
                                 s.params.step_dev), ts):
                dst.copy_(src)
            s.params.latest, s.params.step = latest, step
        del saved
        torch.cuda.synchronize(dev)
        keep = []
        for s in self.stages:
            for d in s.slot_buf:
                keep += list(d.values())
            keep += list(s.live.values()) + list(s.grads.values())
            keep += list(getattr(s, "ids", [])) + list(getattr(s, "labels", []))
        self._keepalive = keep
        self._graph_start = [s.params.latest for s in self.stages]
        g = torch.cuda.CUDAGraph()
        n0 = K.INSTR.launches
        with torch.cuda.graph(g, stream=main):
            self._step(self._gids, self._glabels, None)
            self._restore_ring()
        self.graph_launches = K.INSTR.launches - n0  # kernels one replay launches
        self._graph = g

    def _eager_step(self, ids: torch.Tensor, labels: torch.Tensor,
                    events: Optional[list] = None) -> torch.Tensor:
        last_dev = self.stage_dev[-1]
        caller = torch.cuda.current_stream(last_dev)
        # ... and the pipeline's streams wait for whatever the caller's streams
        # did before (e.g. the H2D copy of ids / labels)
        for d, st in self.streams.items():
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(d))
            st.wait_event(ready)
        if len(self.streams) == 1:  # co-located: everything on one stream
            with torch.cuda.stream(next(iter(self.streams.values()))):
                loss = self._step(ids, labels, events)
        else:
            loss = self._step(ids, labels, events)
        # the loss vector is written on the pipeline's streams: the caller's
        # stream waits for it, so reading it there (e.g. .tolist()) is ordered
        done = torch.cuda.Event()
        done.record(self.streams[last_dev])
        caller.wait_event(done)
        return loss

    def _step(self, ids: torch.Tensor, labels: torch.Tensor, events: Optional[list] = None) -> torch.Tensor:
        if self.multi:
            return self._step_streams(ids, labels, events)
        with torch.cuda.stream(self.streams[self.stage_dev[-1]]):
            self.loss.zero_()
        pending: Dict[Tuple[int, int], Dict[str, torch.Tensor]] = {}
        mailbox: Dict[Tuple[int, int], Dict[str, torch.Tensor]] = {}
        for x, kind, j in self.order:
            with self._arena(x - 1):
                self._op_serial(x, kind, j, ids, labels, events, pending, mailbox)
        if self.sync:  # GPipe: one update per stage after the last backward
            for x, s in enumerate(self.stages):
                with torch.cuda.stream(self.streams[self.stage_dev[x]]), self._arena(x):
                    s.optimizer_step()
        return self.loss

    def _op_serial(self, x, kind, j, ids, labels, events, pending, mailbox) -> None:
        s = self.stages[x - 1]
        st = self.streams[self.stage_dev[x - 1]]
        if events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
        if kind == "fwd":
            if x > 1:
                self._deliver_fwd(x, j, mailbox.pop((x, j)))
            s.forward(j, ids=ids[j - 1] if s.needs_ids else None,
                      labels=labels[j - 1] if s.is_last else None,
                      loss_out=self.loss[j - 1:j] if s.is_last else None)
            if x < self.l:
                mailbox[(x + 1, j)] = self._send_fwd(x, j)
        else:
            for tid, gt in pending.pop((x, j), {}).items():
                s.set_recv_grad(tid, gt)
            grads = s.backward(j)
            if x > 1:
                pending[(x - 1, j)] = self._send_bwd(x, grads)
            s.finish_backward(j)
        if events is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(st)
            events.append((x, j, kind, e0, e1))

    def _step_streams(self, ids, labels, events=None) -> torch.Tensor:
        """Co-located stages on their own streams: fork from the device's main
        stream (where the caller's inputs / timing events live), issue the same
        op order, join back at the end."""
        main = self.streams[self.stage_dev[0]]
        with torch.cuda.stream(main):
            self.loss.zero_()
        fork = torch.cuda.Event()
        fork.record(main)
        for st in self.stage_streams:
            st.wait_event(fork)
        pending: Dict[Tuple[int, int], tuple] = {}
        mailbox: Dict[Tuple[int, int], tuple] = {}
        last = None
        for x, kind, j in self.order:
            with self._arena(x - 1):
                last = self._op_streams(x, kind, j, ids, labels, events, pending, mailbox, last)
        if self.sync:
            for x, s in enumerate(self.stages):
                with self._arena(x):
                    s.optimizer_step()
        for st in self.stage_streams:
            join = torch.cuda.Event()
            join.record(st)
            main.wait_event(join)
        return self.loss

    def _op_streams(self, x, kind, j, ids, labels, events, pending, mailbox, last):
        s = self.stages[x - 1]
        st = self.stage_streams[x - 1]
        if self.serialize and last is not None:
            st.wait_event(last)
        if events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
        if kind == "fwd":
            if x > 1:
                msgs, ev = mailbox.pop((x, j))
                st.wait_event(ev)
                with torch.cuda.stream(st):
                    for tid, msg in msgs.items():
                        s.adopt_recv(tid, j, msg)
            s.forward(j, ids=ids[j - 1] if s.needs_ids else None,
                      labels=labels[j - 1] if s.is_last else None,
                      loss_out=self.loss[j - 1:j] if s.is_last else None)
            if x < self.l:
                mailbox[(x + 1, j)] = self._send_fwd_streams(x, j)
        else:
            if (x, j) in pending:
                gts, ev = pending.pop((x, j))
                st.wait_event(ev)
                for tid, gt in gts.items():
                    s.set_recv_grad(tid, gt)
            grads = s.backward(j)
            if x > 1:
                pending[(x - 1, j)] = self._send_bwd_streams(x, grads)
            s.finish_backward(j)
        if events is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(st)
            events.append((x, j, kind, e0, e1))
        if self.serialize:
            last = torch.cuda.Event()
            last.record(st)
        return last

    def report(self, events: list, t_origin: torch.cuda.Event, losses: torch.Tensor,
               wall_us: float) -> RunReport:
        """Turn the timed events of one step into a SimReport-shaped RunReport."""
        torch.cuda.synchronize()
        ev: List[SimEvent] = []
        done = [0] * (self.m + 1)
        for x, j, kind, e0, e1 in events:
            a = int(round(t_origin.elapsed_time(e0) * 1000))
            b = int(round(t_origin.elapsed_time(e1) * 1000))
            ev.append(SimEvent(x, j, kind, a, b))
            if kind == "bwd" and x == 1:
                done[j] = b
        makespan = max(e.end for e in ev) if ev else 0
        # sync reports the whole iteration (simulate.py:143), async the
        # steady-state time per micro-batch (simulate.py:326-336)
        iteration = float(makespan) if self.sync else async_iteration(done, self.l, self.m, makespan)
        busy = [sum(e.end - e.start for e in ev if e.stage == x + 1) for x in range(self.l)]
        bubble = 1.0 - sum(busy) / (self.l * makespan) if makespan > 0 else 0.0
        measured = self.arena_peaks()
        peaks = measured if measured is not None else list(self.static_bytes)
        top = max(peaks) if peaks else 0
        waste = sum(top - p for p in peaks) / (self.l * top) if top > 0 else 0.0
        cap = self.cfg.capacity
        exceeded = tuple(x + 1 for x, p in enumerate(peaks) if cap is not None and p > cap)
        b = self.cfg.micro_batch_size
        return RunReport(
            per_stage_peak=tuple(peaks), iteration_time=iteration, bubble_ratio=bubble,
            waste_ratio=waste, trace=tuple(sorted(ev, key=lambda e: (e.start, e.end, e.stage, e.mb, e.kind))),
            makespan=makespan, capacity_exceeded=exceeded,
            losses=tuple(float(v) for v in losses.tolist()),
            samples_per_s=((b * (self.m if self.sync else 1)) * 1e6 / iteration) if iteration > 0 else 0.0,
            step_time_us=wall_us,
            device_peak_bytes=max(torch.cuda.max_memory_allocated(d) for d in set(self.stage_dev)),
            per_stage_peak_source="measured: stage arena high-water mark" if measured is not None
            else "static")


def run(plan: PartitionPlan, g: ComputationGraph, cfg: RunConfig,
        model: Optional[TransformerConfig] = None, ids: Optional[torch.Tensor] = None,
        labels: Optional[torch.Tensor] = None, steps: int = 1) -> RunReport:
    """Drop-in for simulate(plan, g, cfg): executes `steps` training iterations
    of the plan on B200s and reports the last one (measured)."""
    from .model import PRESETS, synthetic_batch
    if model is None:
        base = g.name.rsplit("_b", 1)[0]
        if base not in PRESETS:
            raise ValueError(f"cannot infer the model of graph {g.name!r}; pass model=")
        model = PRESETS[base]
    pipe = Pipeline(model, g, plan, cfg)
    try:
        rep = _run(pipe, model, cfg, ids, labels, steps)
        if rep is not None and cfg.measure_stage_peaks and pipe.arenas is None:
            rep = _with_measured_peaks(rep, pipe, model, g, plan, cfg)
        return rep
    finally:
        if pipe.arenas is not None:  # the stages' arenas do not outlive the run
            arenas = pipe.arenas
            del pipe
            K.release_workspaces()  # scratch buffers cached per stage stream live in the arenas
            for a in arenas:
                a.close()
        elif cfg.capacity is not None:  # the cap does not outlive the run
            for d in set(pipe.stage_dev):
                torch.cuda.set_per_process_memory_fraction(1.0, d)


def _run(pipe: Pipeline, model, cfg: RunConfig, ids, labels, steps: int) -> RunReport:
    from .model import synthetic_batch
    if ids is None:
        ids, labels = synthetic_batch(model, cfg.micro_batches, cfg.micro_batch_size, cfg.seed)
    d0, dl = pipe.stage_dev[0], pipe.stage_dev[-1]
    ids_d = ids.to(torch.device("cuda", d0))
    lab_d = labels.to(torch.device("cuda", dl))
    rep = None
    for _ in range(steps):
        events: list = []
        t0 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        t0.record(pipe.streams[d0])
        losses = pipe.step(ids_d, lab_d, events if cfg.trace else None)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) * 1e6
        rep = pipe.report(events, t0, losses, wall) if cfg.trace else None
    return rep


def _with_measured_peaks(rep: RunReport, pipe: Pipeline, model, g: ComputationGraph,
                         plan: PartitionPlan, cfg: RunConfig) -> RunReport:
    """per_stage_peak := each stage's measured device peak when it runs alone
    on its GPU (its 1F1B op list, w + 1 micro-batches, memopt executed) --
    what the planner's _async_peaks model (simulate.py:298-323) predicts for
    the one-stage-per-GPU deployment; waste_ratio and capacity_exceeded follow."""
    import dataclasses
    from .memprobe import probe_stage
    init = init_params(model, cfg.seed)
    peaks = []
    for x in range(1, pipe.l + 1):
        r = probe_stage(model, g, plan, x, cfg.micro_batch_size, device=pipe.stage_dev[x - 1],
                        micro_batches=pipe.l - x + 2, init=init)
        peaks.append(r["peak_bytes"]["measured"])
    top = max(peaks)
    waste = sum(top - p for p in peaks) / (pipe.l * top) if top > 0 else 0.0
    exceeded = tuple(x + 1 for x, p in enumerate(peaks) if cfg.capacity is not None and p > cfg.capacity)
    return dataclasses.replace(rep, per_stage_peak=tuple(peaks), waste_ratio=waste,
                               capacity_exceeded=exceeded,
                               per_stage_peak_source="measured: each stage alone on its GPU")
