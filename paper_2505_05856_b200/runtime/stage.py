"""Per-stage executor of the fine-grained node graph on one B200.

One `StageExecutor` owns a contiguous node range [lo, hi] of the plan
(`stage_bounds`, partition.py:99-103) and everything that range needs on its
device:

  parameters   flat fp32 master / Adam m / Adam v / grad buffers plus a ring of
               w = l-x+1 bf16 weight versions (1F1B weight stashing: the
               forward of micro-batch j uses the newest version, its backward
               the same one; each backward is followed by an AdamW step that
               writes the next version into the slot the retiring micro-batch
               frees).  w matches `schedule_weight` (balance.py:65-77).
  activations  static per-slot buffers (w slots) for every saved tensor this
               stage reads in its backward; tensors the plan evicts (memopt
               actions) live instead in one forward scratch + one backward
               scratch buffer, with pinned host slots for swaps.
  streams      the compute stream (given) and a copy stream for swaps.

Memopt actions are executed exactly (memopt.py:169-322 decides them):
  swap      D2H on the copy stream right after the producing node's forward
            (or right after receipt, for a boundary input), H2D into the
            backward scratch before the stage's backward;
  recompute the tensor is dropped after the forward and rebuilt at backward
            time by replaying exactly `producer_chain` (memopt.py:91-115).

All compute goes through `kernels` -> `_dawnpiper.so`; nothing here computes
with torch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Set, Tuple

import torch

from .. import kernels as K
from ..planner.balance import SCHEDULE_ASYNC, SCHEDULE_SYNC
from ..planner.memplan import MemOptPlan, producer_chain
from ..planner.profile import ComputationGraph
from .graph import internal_tid, out_tid, stats_tid
from .model import (AdamWConfig, NodeDef, TransformerConfig, backward_readers, has_stats,
                    internal_specs, node_rows,
                    output_spec, saved_for_backward)

BF16 = torch.bfloat16
F32 = torch.float32


def _align8(n: int) -> int:
    return (n + 7) // 8 * 8


@dataclass
class ParamSlot:
    name: str
    shape: Tuple[int, ...]
    offset: int
    numel: int
    dense: bool  # gradient fully written by a GEMM (no zeroing / accumulation)


class FlatParams:
    """Flat parameter storage for one stage (master/m/v/grad fp32 + bf16 ring)."""

    def __init__(self, nodes: Sequence[NodeDef], init: Dict[str, torch.Tensor], versions: int,
                 device):
        dense, accum = [], []
        for n in nodes:
            for pn, shp in n.params:
                name = f"{n.id}.{pn}"
                is_dense = ((n.kind in ("linear", "linear_res", "head", "pw", "stem") and pn == "weight")
                            or (n.kind == "xattn" and pn in ("q_weight", "kv_weight")))
                (dense if is_dense else accum).append((name, tuple(shp)))
        self.slots: Dict[str, ParamSlot] = {}
        off = 0
        for group, is_dense in ((dense, True), (accum, False)):
            if not is_dense:
                self.accum_start = off
            for name, shp in group:
                numel = math.prod(shp)
                self.slots[name] = ParamSlot(name, shp, off, numel, is_dense)
                off += _align8(numel)
        self.total = max(8, off)
        self.accum_bytes = (self.total - self.accum_start) * 4
        self.master = torch.zeros(self.total, dtype=F32, device=device)
        for name, s in self.slots.items():
            self.master[s.offset:s.offset + s.numel].copy_(init[name].reshape(-1))
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.grad = torch.zeros_like(self.master)
        self.ring = torch.empty(versions, self.total, dtype=BF16, device=device)
        for k in range(versions):
            K.cast_f32_bf16(self.master, self.ring[k])
        self.step = 0
        # device-resident step count (CUDA-graph mode: the update reads it on
        # the GPU, so a replayed step applies the right bias corrections)
        self.device_step = False
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=device)
        # weight-version ring bookkeeping (PipeDream stashing): the newest
        # version sits in `latest`; micro-batches in flight pin the slot their
        # forward read until their backward retires
        self._build_views()
        self.latest = 0
        self.users: List[Set[int]] = [set() for _ in range(versions)]
        self.version_of: Dict[int, int] = {}

    def pin_latest(self, mb: int) -> int:
        self.version_of[mb] = self.latest
        self.users[self.latest].add(mb)
        return self.latest

    def pinned(self, mb: int) -> int:
        return self.version_of[mb]

    def retire(self, mb: int) -> int:
        """Unpin mb's version; return the slot the next version may overwrite."""
        v = self.version_of.pop(mb)
        self.users[v].discard(mb)
        if not self.users[v]:
            return v
        for k, u in enumerate(self.users):
            if not u:
                return k
        raise RuntimeError("weight-version ring exhausted (more micro-batches in flight than slots)")

    def weight(self, version_slot: int, name: str) -> torch.Tensor:
        return self._wviews[version_slot][name]

    def gradv(self, name: str) -> torch.Tensor:
        return self._gviews[name]

    def _build_views(self) -> None:
        # views are created once: the per-call slicing showed up in host profiles
        self._wviews = [{n: self.ring[k, s.offset:s.offset + s.numel].view(s.shape)
                         for n, s in self.slots.items()} for k in range(self.ring.shape[0])]
        self._gviews = {n: self.grad[s.offset:s.offset + s.numel].view(s.shape)
                        for n, s in self.slots.items()}

    def master_view(self, name: str) -> torch.Tensor:
        s = self.slots[name]
        return self.master[s.offset:s.offset + s.numel].view(s.shape)

    def zero_accum_grads(self, stream=None) -> None:
        if self.accum_bytes:
            K.memset(self.grad[self.accum_start:], 0, self.accum_bytes, stream=stream)

    def adamw(self, out_slot: int, opt: AdamWConfig, stream=None) -> None:
        self.step += 1
        if self.device_step:
            K.adamw_dstep(self.master, self.m, self.v, self.grad, self.ring[out_slot], opt.lr,
                          opt.beta1, opt.beta2, opt.eps, opt.weight_decay, self.step_dev,
                          stream=stream)
        else:
            K.adamw(self.master, self.m, self.v, self.grad, self.ring[out_slot], opt.lr, opt.beta1,
                    opt.beta2, opt.eps, opt.weight_decay, self.step, stream=stream)
        self.latest = out_slot


class StageExecutor:
    def __init__(self, *, cfg: TransformerConfig, g: ComputationGraph, nodes: Sequence[NodeDef],
                 lo: int, hi: int, stage: int, stages: int, micro_batch: int, memopt: MemOptPlan,
                 init: Dict[str, torch.Tensor], device: torch.device, stream: torch.cuda.Stream,
                 opt: AdamWConfig = AdamWConfig(), slots: Optional[int] = None,
                 schedule: str = SCHEDULE_ASYNC, micro_batches: Optional[int] = None,
                 dp_replicas: int = 1):
        self.cfg, self.g = cfg, g
        self.all_nodes = list(nodes)
        self.nodes = self.all_nodes[lo:hi + 1]
        self.lo, self.hi = lo, hi
        self.stage, self.stages = stage, stages
        self.b = micro_batch
        self.M = micro_batch * cfg.seq
        # token rows of the id input (encoder-decoder: src then tgt) and of the head
        self.in_rows = micro_batch * cfg.in_tokens
        self.out_rows = micro_batch * cfg.out_tokens
        self.id_offset = {"embed": 0, "dembed": self.M}
        self.device = device
        self.stream = stream
        # swap engine: one copy stream per direction, so a micro-batch's D2H
        # offloads and an earlier micro-batch's H2D prefetches use both
        # directions of the host link at once (1F1B interleaves them)
        self.copy_stream = torch.cuda.Stream(device=device)      # D2H
        self.h2d_stream = torch.cuda.Stream(device=device)       # H2D
        self.d2h_done: Dict[Tuple[str, int], torch.cuda.Event] = {}
        self.opt = opt
        if schedule not in (SCHEDULE_ASYNC, SCHEDULE_SYNC):
            raise ValueError(f"unknown schedule {schedule!r}")
        # GPipe (sync, simulate.py:169-208): every micro-batch of the iteration is
        # in flight before the first backward (schedule_weight = m,
        # balance.py:65-77), one weight version, gradients accumulated over the
        # m micro-batches and one AdamW step at the end of the iteration
        self.sync = schedule == SCHEDULE_SYNC
        if self.sync and micro_batches is None and slots is None:
            raise ValueError("the sync schedule needs micro_batches")
        self.m_sync = micro_batches if self.sync else 1
        if slots is not None:
            self.w = slots
        else:
            self.w = micro_batches if self.sync else stages - stage + 1
        # dense weight gradients are written by the first backward of an
        # iteration and accumulated by the rest (sync only)
        self._wgrad_acc = False
        # mean over the iteration's tokens (and, with data-parallel replicas whose
        # gradients are summed by an all-reduce, over the replicas)
        self.dp_replicas = dp_replicas
        self.grad_scale = 1.0 / (self.out_rows * self.m_sync * dp_replicas)
        self.is_first = lo == 0
        # stages holding an embedding node take the micro-batch's token ids
        # (encoder-decoder: `dembed` may sit behind a cut at position 0)
        self.needs_ids = any(n.kind in ("embed", "stem") for n in self.nodes)
        self.cnn = getattr(cfg, "family", "transformer") == "cnn"
        # gradient buffers shared by the two inputs of an `add` (CNN graphs copy
        # one on the first in-place accumulation into it)
        self.shared_grads: Set[str] = set()
        self.is_last = hi == len(self.all_nodes) - 1
        self.node_by_id = {n.id: n for n in self.all_nodes}
        self.index = {n.id: i for i, n in enumerate(self.all_nodes)}
        self.params = FlatParams(self.nodes, init, 1 if self.sync else self.w, device)

        # ---- tensor bookkeeping -------------------------------------------------
        self.readers = backward_readers(self.all_nodes)
        in_stage = {n.id for n in self.nodes}
        # boundary inputs: outputs of earlier stages consumed here or relayed onward
        self.recv_ids = self._boundary(lo - 1) if not self.is_first else []
        self.send_ids = self._boundary(hi) if not self.is_last else []
        # tensors some backward in this stage reads
        needed: Set[str] = set()
        for n in self.nodes:
            needed.update(self.self_tids(n))
        for src, rd in self.readers.items():
            if any(r in in_stage for r in rd) and saved_for_backward(self.node_by_id[src]):
                needed.add(out_tid(src))
        self.needed = needed
        acts = {a.tensor_id: a for a in memopt.actions}
        self.swap_ids = {t for t, a in acts.items() if a.kind == "swap"}
        self.recompute_ids = {t for t, a in acts.items() if a.kind == "recompute"}
        unknown = (self.swap_ids | self.recompute_ids) - needed
        if unknown:
            raise ValueError(f"stage {stage}: memopt names tensors it does not hold: {sorted(unknown)}")
        # recompute chains (memopt.py:91-115), replayed in forward order.  What a
        # chain reads from outside itself must still be there at backward time:
        # the chain stops at saved tensors inside the stage, but a boundary
        # tensor received from the previous stage can feed it directly, so such
        # inputs are kept resident like saved tensors.
        self.chains: Dict[str, List[int]] = {}
        for tid in sorted(self.recompute_ids):
            p = self.index[tid.rsplit(".", 1)[0]]
            chain, _ = producer_chain(g, p, lo, hi)
            self.chains[tid] = chain
            inside = {self.all_nodes[i].id for i in chain}
            for i in chain:
                needed.update(out_tid(u) for u in self.all_nodes[i].inputs if u not in inside)

        # Residency classes: resident saved tensors get one static buffer per
        # in-flight slot; evicted tensors (memopt actions) are allocated only
        # while alive -- from production until their last in-stage forward
        # reader (and their D2H, for swaps), and from a just-in-time swap-in /
        # recompute before their first backward reader until their last -- so
        # they cost no device memory in between (the planner's
        # w * (micro_peak - saved) model, memopt.py:156-158); transient
        # un-saved tensors ("ephemeral") live the same way, from production to
        # their last in-stage forward reader (the m_d release of the profile,
        # runtime/graph.py), never across micro-batches.
        self.evicted = self.swap_ids | self.recompute_ids
        self.slot_buf: List[Dict[str, torch.Tensor]] = [{} for _ in range(self.w)]
        self.ephemeral: Set[str] = set()
        self.host: Dict[str, List[torch.Tensor]] = {}
        self.live: Dict[str, torch.Tensor] = {}
        ids_needed = {out_tid(n) for n in self._produced_or_received()}
        ids_needed |= {t for n in self.nodes for t in self.self_tids(n)}
        for tid in sorted(ids_needed):
            shape, dt = self._spec(tid)
            if tid in needed and tid not in self.evicted:
                for k in range(self.w):
                    self.slot_buf[k][tid] = torch.empty(shape, dtype=dt, device=device)
            elif tid in needed:
                if tid in self.swap_ids:
                    self.host[tid] = [torch.empty(shape, dtype=dt, pin_memory=True)
                                      for _ in range(self.w)]
            else:
                self.ephemeral.add(tid)
        if self.needs_ids:
            ishape, idt = cfg.input_spec(micro_batch)
            self.ids = [torch.empty(ishape, dtype=idt, device=device) for _ in range(self.w)]
        if self.is_last:
            self.labels = [torch.empty(self.out_rows, dtype=torch.int32, device=device)
                           for _ in range(self.w)]
            self.loss = torch.zeros(1, dtype=F32, device=device)
        self.swap_in_done: Dict[str, torch.cuda.Event] = {}
        # D2H back-pressure: memory of a swapped tensor is recycled only once its
        # D2H completes; if the host link falls behind compute, the forward
        # waits for the oldest transfer instead of piling up device memory
        self.d2h_pending: List[Tuple[torch.cuda.Event, int]] = []
        # bytes of swapped tensors whose D2H is still in flight: device memory the
        # planner's model does not see (memopt.py:156-158 frees a swapped tensor
        # at once); 256 MiB is ~5 ms of the measured 55 GB/s host link
        self.d2h_budget = 256 << 20
        # per-slot micro-batch bookkeeping
        self.slot_mb = [0] * self.w
        self.grads: Dict[str, torch.Tensor] = {}
        self.grad_init: Set[str] = set()
        self.recv_grads: Dict[str, torch.Tensor] = {}
        # GELU fused into its neighbours' GEMM epilogues when fc1 -> gelu -> fc2
        # live in this stage: fc1's forward writes f (aux) and gelu(f); fc2's
        # dgrad writes df = (dz W2) * gelu'(f) straight into f's gradient.
        self.fwd_gelu_of: Dict[str, str] = {}   # fc1 id -> gelu id
        self.bwd_gelu_of: Dict[str, str] = {}   # fc2 id -> gelu id
        for n in self.nodes:
            if n.kind == "gelu" and n.inputs[0] in in_stage:
                src = self.node_by_id[n.inputs[0]]
                if src.kind == "linear":
                    self.fwd_gelu_of[src.id] = n.id
                users = [c for c in self.nodes if n.id in c.inputs]
                if len(users) == 1 and users[0].kind == "linear":
                    self.bwd_gelu_of[users[0].id] = n.id
        # fc1's bias gradient folded into fc2's dgrad epilogue (dpn_gemm colsum):
        # df written there is fc1's complete output gradient when the GELU is the
        # only reader of fc1's output anywhere in the graph
        self.gelu_bias_of: Dict[str, str] = {}  # fc2 id -> fc1 id
        for fc2_id, g_id in self.bwd_gelu_of.items():
            src = self.node_by_id[g_id].inputs[0]
            if (src in in_stage and self.node_by_id[src].kind == "linear"
                    and [c.id for c in self.all_nodes if src in c.inputs] == [g_id]):
                self.gelu_bias_of[fc2_id] = src
        # QKV bias gradient accumulated by the fused attention backward
        self.attn_bias_of: Dict[str, str] = {}  # attention id -> qkv linear id
        for n in self.nodes:
            if n.kind == "attn_fused" and n.inputs[0] in in_stage:
                src = self.node_by_id[n.inputs[0]]
                if (src.kind == "linear"
                        and [c.id for c in self.all_nodes if src.id in c.inputs] == [n.id]):
                    self.attn_bias_of[n.id] = src.id
        self._skip_bwd: Set[str] = set()
        # bias gradient of a linear node folded into the one-pass LayerNorm
        # backward of the LN reading that node's output (or, through the
        # residual `add`, fc2's): the LN's final dx IS the linear's output
        # gradient when the LN is the lowest-index in-stage consumer (every
        # other contribution has landed), so its column sums are the bias
        # gradient and the separate colsum pass over dy is skipped
        self.ln_bias_of: Dict[str, str] = {}
        self._bias_done: Set[str] = set()
        spos = {n.id: i for i, n in enumerate(self.nodes)}
        for n in self.nodes:
            if n.kind != "ln" or n.inputs[0] not in in_stage:
                continue
            u = self.node_by_id[n.inputs[0]]
            lin = u
            if u.kind == "add" and u.inputs[0] in in_stage:
                lin = self.node_by_id[u.inputs[0]]
                if lin.kind != "linear":
                    continue
            elif u.kind not in ("linear", "linear_res"):
                continue
            if not any(pn == "bias" for pn, _ in lin.params):
                continue
            first = min(spos[c.id] for c in self.nodes if u.id in c.inputs)
            if first == spos[n.id]:
                self.ln_bias_of[n.id] = lin.id
        # residual add fused into fc2's epilogue when both live in this stage:
        # fc2's forward writes z + y straight into the add node's output
        # (fc2's own output z is never materialised: nothing reads it later)
        self.fwd_add_of: Dict[str, str] = {}    # fc2 id -> add id
        recv_nodes = {t.rsplit(".", 1)[0] for t in self.recv_ids}
        for n in self.nodes:
            if n.kind == "add" and n.inputs[0] in in_stage and (
                    n.inputs[1] in in_stage or n.inputs[1] in recv_nodes):
                src = self.node_by_id[n.inputs[0]]
                if (src.kind == "linear" and not saved_for_backward(src)
                        and out_tid(src.id) not in self.send_ids):
                    self.fwd_add_of[src.id] = n.id
        # lifetimes of evicted tensors (positions within this stage's node list)
        pos = {n.id: i for i, n in enumerate(self.nodes)}
        self.fwd_last: Dict[str, float] = {}
        for tid in self.evicted | self.ephemeral:
            src, kind = tid.rsplit(".", 1)
            users = [src] if kind != "out" else [n.id for n in self.nodes if src in n.inputs]
            last = max((pos[u] for u in users), default=-1)
            self.fwd_last[tid] = math.inf if tid in self.send_ids else last
        self.bwd_reads: Dict[str, List[str]] = {}
        for n in self.nodes:
            reads = [out_tid(src) for src, rd in self.readers.items() if n.id in rd]
            reads += self.self_tids(n)
            if n.id in self.bwd_gelu_of:  # fused GELU backward reads the pre-activation
                reads.append(out_tid(self.node_by_id[self.bwd_gelu_of[n.id]].inputs[0]))
            self.bwd_reads[n.id] = [t for t in reads if t in self.evicted]
        self.bwd_last: Dict[str, int] = {}
        self.bwd_first: Dict[str, int] = {}
        for n in self.nodes:
            for t in self.bwd_reads[n.id]:
                self.bwd_last[t] = min(self.bwd_last.get(t, pos[n.id]), pos[n.id])
                self.bwd_first[t] = max(self.bwd_first.get(t, pos[n.id]), pos[n.id])
        self.swap_lookahead = 2
        # early prefetch: at the end of micro-batch mb's backward, H2D of up to
        # this many bytes of mb+1's swapped tensors starts, so it overlaps the
        # next forward's D2H offloads (1F1B runs F(mb+w) between B(mb) and
        # B(mb+1)); the bytes are held that much earlier than just-in-time
        self.prefetch_budget = 0
        self.prefetched: Dict[str, Tuple[torch.Tensor, torch.cuda.Event]] = {}
        self._recv_mb = 0  # micro-batch whose boundary inputs are being delivered
        # profiler hook: when a list, every node forward / backward is bracketed
        # with CUDA events on the compute stream -> (node id, "fwd"|"bwd", e0, e1)
        self.node_timer: Optional[list] = None
        # memory-plan instrumentation: when a dict of lists, the swap engine and
        # recompute replay record timing events -- "d2h" / "h2d": (bytes, start,
        # end) on the copy stream; "stall": compute-stream waits on a swap-in;
        # "recompute": replayed producer chains (runtime/memprobe.py)
        self.memstats: Optional[Dict[str, list]] = None

    # ---- helpers -------------------------------------------------------------------

    def self_tids(self, n: NodeDef) -> List[str]:
        """Tensors n produces besides its output that only its own backward reads:
        statistics (LayerNorm mean/rstd, attention LSE) and internal tensors
        (cross-attention q / kv / P)."""
        out = [stats_tid(n.id)] if has_stats(n) else []
        return out + [internal_tid(n.id, k) for k in internal_specs(self.cfg, n, self.b)]

    def _boundary(self, pos: int) -> List[str]:
        """Output tids crossing the cut after canonical index pos (simulate.py:93-100)."""
        last = self.g.last_consumer
        return [out_tid(self.all_nodes[u].id) for u in range(pos + 1) if last[u] > pos]

    def _produced_or_received(self) -> List[str]:
        ids = [n.id for n in self.nodes]
        ids += [t.rsplit(".", 1)[0] for t in self.recv_ids]
        return ids

    def _spec(self, tid: str):
        nid, kind = tid.rsplit(".", 1)
        node = self.node_by_id[nid]
        if kind == "stats":
            if node.kind == "bn":
                return (2, dict(node.attrs)["C"]), F32
            if node.kind == "attn_fused":
                return (self.b, self.cfg.heads, node.seq or self.cfg.seq), F32
            return (2, node_rows(self.cfg, node, self.b)), F32
        if kind != "out":
            return internal_specs(self.cfg, node, self.b)[kind]
        return output_spec(self.cfg, node, self.b)

    def buf(self, tid: str, slot: int, phase: str) -> torch.Tensor:
        if tid in self.slot_buf[slot]:
            return self.slot_buf[slot][tid]
        if tid in self.evicted or tid in self.ephemeral:
            if tid not in self.live:
                raise KeyError(f"stage {self.stage}: tensor {tid} is not materialised")
            return self.live[tid]
        raise KeyError(f"stage {self.stage}: no buffer for {tid}")

    def _alloc_live(self, tid: str) -> torch.Tensor:
        # callers run inside `with torch.cuda.stream(self.stream)` (forward /
        # backward / the schedulers), so allocations are compute-stream ordered
        shape, dt = self._spec(tid)
        t = torch.empty(shape, dtype=dt, device=self.device)
        self.live[tid] = t
        return t

    def _drop_leftovers(self) -> None:
        """Release evicted tensors a previous forward kept only for its sends."""
        for t in [t for t in self.live if self.fwd_last.get(t) == math.inf]:
            del self.live[t]

    def _begin_recv(self, mb: int) -> None:
        """First delivery of micro-batch mb: the previous forward's send-only
        leftovers go now, once -- not per delivered tensor, which would drop a
        relayed tensor of mb itself delivered earlier in the same batch."""
        if self._recv_mb != mb:
            self._drop_leftovers()
            self._recv_mb = mb

    def slot_of(self, mb: int) -> int:
        return (mb - 1) % self.w


    # ---- forward -------------------------------------------------------------------

    def forward(self, mb: int, ids: Optional[torch.Tensor] = None,
                labels: Optional[torch.Tensor] = None, loss_out: Optional[torch.Tensor] = None) -> None:
        """Forward of micro-batch mb (1-based).  Boundary inputs must already be in
        `recv_buffer(tid, mb)`; ids/labels are device int32 [M] for the first/last stage."""
        st = self.stream
        slot = self.slot_of(mb)
        self.slot_mb[slot] = mb
        ver = self.params.pin_latest(mb)
        with torch.cuda.stream(st):
            if self.needs_ids:
                self.ids[slot].copy_(ids, non_blocking=True)
            if self.is_last:
                self.labels[slot].copy_(labels, non_blocking=True)
            for tid in self.recv_ids:
                if tid in self.swap_ids:
                    self._swap_out(tid, slot)
                if (tid in self.evicted or tid in self.ephemeral) and self.fwd_last[tid] < 0:
                    del self.live[tid]
            fused_gelus = set(self.fwd_gelu_of.values()) | set(self.fwd_add_of.values())
            for i, n in enumerate(self.nodes):
                produced = [] if n.id in fused_gelus else self._outputs(n)  # fused: fc1 made it
                if any(t in self.swap_ids for t in produced):
                    self._d2h_backpressure()
                for t in produced:
                    if t in self.evicted or t in self.ephemeral:
                        self._alloc_live(t)
                if self.node_timer is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                self._node_fwd(n, slot, ver, "fwd", loss_out)
                if self.node_timer is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(st)
                    self.node_timer.append((n.id, "fwd", e0, e1))
                for t in produced:
                    if t in self.swap_ids:
                        self._swap_out(t, slot)
                for t in [t for t in self.live if self.fwd_last.get(t, math.inf) <= i]:
                    del self.live[t]  # last in-stage forward reader done (swaps: D2H ordered)

    def recv_buffer(self, tid: str, mb: int) -> torch.Tensor:
        if tid in self.evicted or tid in self.ephemeral:
            self._begin_recv(mb)
            return self._alloc_live(tid)
        return self.buf(tid, self.slot_of(mb), "fwd")

    def recv_like(self, tid: str) -> torch.Tensor:
        """A fresh device buffer shaped like boundary input tid (an early-posted
        receive lands in it; `adopt_recv` then takes it over)."""
        shape, dt = self._spec(tid)
        return torch.empty(shape, dtype=dt, device=self.device)

    def adopt_recv(self, tid: str, mb: int, msg: torch.Tensor) -> None:
        """Zero-copy receive (co-located stages): the message buffer becomes this
        stage's buffer of tid for micro-batch mb.  The sender hands over a
        private copy, so nothing else writes it."""
        if tid in self.evicted or tid in self.ephemeral:
            self._begin_recv(mb)
            self.live[tid] = msg
            return
        slot = self.slot_of(mb)
        if tid in self.slot_buf[slot]:
            self.slot_buf[slot][tid] = msg
        else:
            raise KeyError(f"stage {self.stage}: no buffer for {tid}")

    def send_buffer(self, tid: str, mb: int) -> torch.Tensor:
        return self.buf(tid, self.slot_of(mb), "fwd")

    def release_send_buffer(self, tid: str, mb: int) -> Optional[torch.Tensor]:
        """Give away this stage's buffer of boundary tensor tid for micro-batch mb
        (co-located zero-copy send) when the stage's own backward never reads it;
        a fresh buffer takes its place.  None when it must be copied instead."""
        if tid in self.needed or tid in self.evicted:
            return None
        slot = self.slot_of(mb)
        if tid in self.slot_buf[slot]:
            t = self.slot_buf[slot][tid]
            self.slot_buf[slot][tid] = torch.empty_like(t)
            return t
        if tid in self.ephemeral and tid in self.live:
            return self.live.pop(tid)
        return None

    def _outputs(self, n: NodeDef) -> List[str]:
        outs = [out_tid(n.id)] + self.self_tids(n)
        if n.id in self.fwd_gelu_of:
            outs.append(out_tid(self.fwd_gelu_of[n.id]))
        if n.id in self.fwd_add_of:
            outs.append(out_tid(self.fwd_add_of[n.id]))
        return outs

    def _swap_out(self, tid: str, slot: int) -> None:
        """D2H of an evicted tensor on the copy stream (swap engine, memopt swap),
        through the C-ABI's dpn_swap_out: the copy stream waits on an event of
        the compute stream, so the copy reads the finished tensor."""
        ev = torch.cuda.Event()
        ev.record(self.stream)
        cs = self.copy_stream
        src = self.live[tid]
        t0 = self._stat_event(cs, ev)
        nbytes = K.swap_out(self.host[tid][slot], src, cs, ready_event=ev)
        src.record_stream(cs)  # memory is recycled only after the D2H completes
        done = torch.cuda.Event(enable_timing=self.memstats is not None)
        done.record(cs)
        if self.memstats is not None:
            self.memstats["d2h"].append((nbytes, t0, done))
        self.d2h_pending.append((done, nbytes))
        self.d2h_done[(tid, slot)] = done  # the H2D of this slot reads after it

    def _stat_event(self, stream, after=None):
        """A timing event on `stream` (after `after`) when memstats is on."""
        if self.memstats is None:
            return None
        if after is not None:
            stream.wait_event(after)
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def _d2h_backpressure(self) -> None:
        while self.d2h_pending and sum(b for _, b in self.d2h_pending) > self.d2h_budget:
            ev, _ = self.d2h_pending.pop(0)
            self.stream.wait_event(ev)

    def _swap_in(self, tid: str, slot: int, early: bool = False) -> None:
        """H2D prefetch of a swapped tensor into a fresh device buffer (early:
        held in `prefetched` until its micro-batch's backward starts)."""
        if early:
            shape, dt = self._spec(tid)
            dst = torch.empty(shape, dtype=dt, device=self.device)
        else:
            dst = self._alloc_live(tid)
        ev = torch.cuda.Event()
        ev.record(self.stream)  # the buffer's memory is free in compute-stream order
        cs = self.h2d_stream
        written = self.d2h_done.pop((tid, slot), None)
        if written is not None:  # the host slot holds this micro-batch's copy
            cs.wait_event(written)
        t0 = self._stat_event(cs, ev)
        nbytes = K.swap_in(dst, self.host[tid][slot], cs, ready_event=ev)
        done = torch.cuda.Event(enable_timing=self.memstats is not None)
        done.record(cs)
        if self.memstats is not None:
            self.memstats["h2d"].append((nbytes, t0, done))
        if early:
            self.prefetched[tid] = (dst, done)
        else:
            self.swap_in_done[tid] = done

    def _node_fwd(self, n: NodeDef, slot: int, ver: int, phase: str,
                  loss_out: Optional[torch.Tensor] = None) -> None:
        cfg, M, H = self.cfg, self.M, self.cfg.hidden
        st = self.stream
        W = lambda pn: self.params.weight(ver, f"{n.id}.{pn}")
        out = self.buf(out_tid(n.id), slot, phase)
        inp = [self.buf(out_tid(u), slot, phase) for u in n.inputs]
        k = n.kind
        if k == "embed":
            off, rows = self.id_offset[n.id], node_rows(cfg, n, self.b)
            K.embed_fwd(self.ids[slot][off:off + rows], W("tok"), W("pos"), out, n.seq or cfg.seq,
                        stream=st)
        elif k == "ln":
            stats = self.buf(stats_tid(n.id), slot, phase)
            K.layernorm_fwd(inp[0], W("gamma"), W("beta"), out, stats[0], stats[1], cfg.ln_eps,
                            stream=st)
        elif k == "linear":
            g_id = self.fwd_gelu_of.get(n.id) if phase == "fwd" else None
            a_id = self.fwd_add_of.get(n.id) if phase == "fwd" else None
            if g_id is not None:  # out = f (pre-activation), gelu node's buffer = gelu(f)
                K.linear_fwd(inp[0], W("weight"), self.buf(out_tid(g_id), slot, phase),
                             bias=W("bias"), gelu=True, aux=out, stream=st)
            elif a_id is not None:  # add node's buffer = x W^T + b + residual
                a = self.node_by_id[a_id]
                K.linear_fwd(inp[0], W("weight"), self.buf(out_tid(a_id), slot, phase),
                             bias=W("bias"), residual=self.buf(out_tid(a.inputs[1]), slot, phase),
                             stream=st)
            else:
                K.linear_fwd(inp[0], W("weight"), out, bias=W("bias"), stream=st)
        elif k == "linear_res":
            K.linear_fwd(inp[0], W("weight"), out, bias=W("bias"), residual=inp[1], stream=st)
        elif k == "gelu":
            if not (phase == "fwd" and n.inputs[0] in self.fwd_gelu_of):
                K.gelu_fwd(inp[0], out, stream=st)
        elif k == "add":
            if not (phase == "fwd" and n.inputs[0] in self.fwd_add_of):
                K.add(inp[0], inp[1], out, stream=st)
        elif k == "score":
            self._scores(inp[0], out, n.seq or cfg.seq)
            K.softmax_fwd(out, out, n.seq or cfg.seq, 1.0 / math.sqrt(cfg.head_dim), n.causal,
                          stream=st)
        elif k == "attn":
            self._pv(inp[0], inp[1], out, n.seq or cfg.seq)
        elif k == "attn_fused":
            lse = self.buf(stats_tid(n.id), slot, phase)
            K.attn_fwd(inp[0], out, lse, self.b, n.seq or cfg.seq, cfg.heads, n.causal, stream=st)
        elif k == "xattn":
            self._xattn_fwd(n, inp[0], inp[1], out, slot, phase, W)
        elif k == "head":
            K.linear_fwd(inp[0], W("weight"), out, stream=st)
            # fused loss + dlogits; on a recompute replay the loss is discarded
            loss = (loss_out if loss_out is not None else self.loss) if phase == "fwd" else self._scratch_loss()
            K.xent(out, self.labels[slot], cfg.vocab, self.grad_scale, loss, out,
                   loss_scale=1.0 / self.out_rows, stream=st)
        elif self.cnn:
            self._cnn_fwd(n, inp, out, slot, phase, W)
        else:
            raise ValueError(k)

    # ---- CNN nodes (runtime/cnn.py) -------------------------------------------------

    def _stem_cols(self, n: NodeDef, slot: int) -> torch.Tensor:
        a, b = dict(n.attrs), self.b
        cols = torch.empty(b * a["Ho"] * a["Wo"], 9 * a["Cin"], dtype=BF16, device=self.device)
        K.im2col3(self.ids[slot], cols, b, a["H"], a["W"], a["Cin"], a["stride"], stream=self.stream)
        return cols

    def _cnn_fwd(self, n: NodeDef, inp, out, slot: int, phase: str, W) -> None:
        st, b, k = self.stream, self.b, n.kind
        a = dict(n.attrs)
        if k == "stem":
            K.linear_fwd(self._stem_cols(n, slot), W("weight"), out, stream=st)
        elif k == "bn":
            K.bn_fwd(inp[0], W("gamma"), W("beta"), out, self.buf(stats_tid(n.id), slot, phase),
                     self.cfg.bn_eps, stream=st)
        elif k == "relu":
            K.relu_fwd(inp[0], out, stream=st)
        elif k == "pw":
            K.linear_fwd(inp[0], W("weight"), out, stream=st)
        elif k == "dw":
            K.dwconv3_fwd(inp[0], W("weight"), out, b, a["H"], a["W"], a["C"], a["stride"], stream=st)
        elif k == "pool":
            arg = self.buf(internal_tid(n.id, "arg"), slot, phase) if a["mode"] == 0 else None
            K.pool3_fwd(inp[0], out, arg, b, a["H"], a["W"], a["C"], a["stride"], a["mode"], stream=st)
        elif k == "concat":
            off, P = 0, out.shape[0]
            for x in inp:
                K.copy_cols(x, x.shape[1], out[:, off:], out.shape[1], P, x.shape[1], stream=st)
                off += x.shape[1]
        elif k == "gap":
            K.gap_fwd(inp[0], out, b, a["H"] * a["W"], a["C"], stream=st)
        else:
            raise ValueError(k)

    def _own(self, tid: str) -> torch.Tensor:
        """grads[tid] for an in-place update: a buffer still shared with another
        tensor's gradient is copied first."""
        if tid in self.shared_grads:
            self.grads[tid] = self.grads[tid].clone()
            self.shared_grads.discard(tid)
        return self.grads[tid]

    def _dx_target(self, x_t: str):
        """Where a node writes its contribution to x_t's gradient: the gradient
        buffer itself on first contribution, else a temporary to be added."""
        if x_t not in self.grad_init:
            buf = self.grad_buffer(x_t)
            self.grad_init.add(x_t)
            return buf, False
        return self.grad_like(x_t), True

    def _dx_done(self, x_t: str, t: torch.Tensor, pending: bool) -> None:
        if pending:
            dst = self._own(x_t)
            K.add(dst, t, dst, stream=self.stream)

    def _cnn_bwd(self, n: NodeDef, dy, slot: int, W, G) -> None:
        st, b, k = self.stream, self.b, n.kind
        a = dict(n.attrs)
        if k == "stem":  # the images need no gradient: weight gradient only
            K.linear_wgrad(dy, self._stem_cols(n, slot), G("weight"), accumulate=self._wgrad_acc,
                           stream=st)
            return
        if k == "concat":
            off = 0
            for u in n.inputs:
                t = out_tid(u)
                C = self._spec(t)[0][1]
                if t not in self.grad_init:
                    dst = self.grad_buffer(t)
                    self.grad_init.add(t)
                    K.copy_cols(dy[:, off:], dy.shape[1], dst, C, dy.shape[0], C, stream=st)
                else:
                    K.copy_cols(dy[:, off:], dy.shape[1], self._own(t), C, dy.shape[0], C,
                                accumulate=True, stream=st)
                off += C
            return
        x_t = out_tid(n.inputs[0])
        if k == "pw":
            x = self.buf(x_t, slot, "bwd")
            if x_t in self.grad_init:
                dx = self._own(x_t)
                K.linear_dgrad(dy, W("weight"), dx, accumulate_into=dx, stream=st)
            else:
                K.linear_dgrad(dy, W("weight"), self.grad_buffer(x_t), stream=st)
                self.grad_init.add(x_t)
            K.linear_wgrad(dy, x, G("weight"), accumulate=self._wgrad_acc, stream=st)
            return
        dx, pending = self._dx_target(x_t)
        if k == "bn":
            ws = torch.empty(2 * a["C"], dtype=F32, device=self.device)
            K.bn_bwd(dy, self.buf(x_t, slot, "bwd"), self.buf(stats_tid(n.id), slot, "bwd"),
                     W("gamma"), dx, G("gamma"), G("beta"), ws, self.cfg.bn_eps, stream=st)
        elif k == "relu":
            K.relu_bwd(dy, self.buf(out_tid(n.id), slot, "bwd"), dx, stream=st)
        elif k == "dw":
            K.dwconv3_bwd(self.buf(x_t, slot, "bwd"), W("weight"), dy, dx, G("weight"), b, a["H"],
                          a["W"], a["C"], a["stride"], stream=st)
        elif k == "pool":
            arg = self.buf(internal_tid(n.id, "arg"), slot, "bwd") if a["mode"] == 0 else None
            K.pool3_bwd(dy, arg, dx, b, a["H"], a["W"], a["C"], a["stride"], a["mode"], stream=st)
        elif k == "gap":
            K.gap_bwd(dy, dx, b, a["H"] * a["W"], a["C"], stream=st)
        else:
            raise ValueError(k)
        self._dx_done(x_t, dx, pending)

    def _scratch_loss(self):
        if not hasattr(self, "_sl"):
            self._sl = torch.zeros(1, dtype=F32, device=self.device)
        return self._sl

    # cross-attention (decoder): q from the decoder stream, k/v from E
    def _xattn_fwd(self, n: NodeDef, c, E, out, slot: int, phase: str, W) -> None:
        cfg, st = self.cfg, self.stream
        t, s, d, A, H, b = n.seq, cfg.seq, cfg.head_dim, cfg.heads, cfg.hidden, self.b
        q = self.buf(internal_tid(n.id, "q"), slot, phase)
        kv = self.buf(internal_tid(n.id, "kv"), slot, phase)
        K.linear_fwd(c, W("q_weight"), q, bias=W("q_bias"), stream=st)
        K.linear_fwd(E, W("kv_weight"), kv, bias=W("kv_bias"), stream=st)
        if cfg.fused_attention:  # flash-style cross-attention, P never materialised
            K.attn_fwd_cross(q, kv, out, self.buf(internal_tid(n.id, "lse"), slot, phase), b, t, s, A,
                             stream=st)
            return
        P = self.buf(internal_tid(n.id, "p"), slot, phase)
        # S = q K^T per (batch, head): [t, s]
        K.gemm_raw(M=t, N=s, K=d, A=q, lda=H, a_s=(d, t * H), B=kv, ldb=2 * H, b_s=(d, s * 2 * H),
                   batch1=A, batch2=b, Cout=P, ldc=s, c_s=(t * s, A * t * s), stream=st)
        K.softmax_fwd(P, P, t, 1.0 / math.sqrt(d), False, stream=st)
        # O = P V: V rows are s-contiguous per head (MN-major over d)
        K.gemm_raw(M=t, N=d, K=s, A=P, lda=s, a_s=(t * s, A * t * s), B=kv[:, H:], ldb=2 * H,
                   b_mn=True, b_s=(d, s * 2 * H), batch1=A, batch2=b, Cout=out, ldc=H,
                   c_s=(d, t * H), stream=st)

    def _xattn_bwd(self, n: NodeDef, dy, slot: int, W, G) -> None:
        cfg, st = self.cfg, self.stream
        t, s, d, A, H, b = n.seq, cfg.seq, cfg.head_dim, cfg.heads, cfg.hidden, self.b
        c_t, e_t = out_tid(n.inputs[0]), out_tid(n.inputs[1])
        c, E = self.buf(c_t, slot, "bwd"), self.buf(e_t, slot, "bwd")
        q = self.buf(internal_tid(n.id, "q"), slot, "bwd")
        kv = self.buf(internal_tid(n.id, "kv"), slot, "bwd")
        dq = torch.empty_like(q)
        dkv = torch.empty_like(kv)
        if cfg.fused_attention:
            K.attn_bwd_cross(q, kv, self.buf(out_tid(n.id), slot, "bwd"), dy,
                             self.buf(internal_tid(n.id, "lse"), slot, "bwd"), dq, dkv, b, t, s, A,
                             stream=st)
        else:
            self._xattn_bwd_unfused(n, dy, q, kv, dq, dkv, slot)
        self._xattn_proj_bwd(n, c_t, c, e_t, E, dq, dkv, W, G)

    def _xattn_bwd_unfused(self, n: NodeDef, dy, q, kv, dq, dkv, slot: int) -> None:
        cfg, st = self.cfg, self.stream
        t, s, d, A, H, b = n.seq, cfg.seq, cfg.head_dim, cfg.heads, cfg.hidden, self.b
        P = self.buf(internal_tid(n.id, "p"), slot, "bwd")
        dS = torch.empty_like(P)
        # dP = dO V^T
        K.gemm_raw(M=t, N=s, K=d, A=dy, lda=H, a_s=(d, t * H), B=kv[:, H:], ldb=2 * H,
                   b_s=(d, s * 2 * H), batch1=A, batch2=b, Cout=dS, ldc=s, c_s=(t * s, A * t * s),
                   stream=st)
        # dV = P^T dO
        K.gemm_raw(M=s, N=d, K=t, A=P, lda=s, a_mn=True, a_s=(t * s, A * t * s), B=dy, ldb=H,
                   b_mn=True, b_s=(d, t * H), batch1=A, batch2=b, Cout=dkv[:, H:], ldc=2 * H,
                   c_s=(d, s * 2 * H), stream=st)
        K.softmax_bwd(P, dS, dS, 1.0 / math.sqrt(d), stream=st)  # dS (scale folded)
        # dq = dS K ; dK = dS^T q
        K.gemm_raw(M=t, N=d, K=s, A=dS, lda=s, a_s=(t * s, A * t * s), B=kv, ldb=2 * H, b_mn=True,
                   b_s=(d, s * 2 * H), batch1=A, batch2=b, Cout=dq, ldc=H, c_s=(d, t * H), stream=st)
        K.gemm_raw(M=s, N=d, K=t, A=dS, lda=s, a_mn=True, a_s=(t * s, A * t * s), B=q, ldb=H,
                   b_mn=True, b_s=(d, t * H), batch1=A, batch2=b, Cout=dkv, ldc=2 * H,
                   c_s=(d, s * 2 * H), stream=st)

    def _xattn_proj_bwd(self, n: NodeDef, c_t, c, e_t, E, dq, dkv, W, G) -> None:
        st = self.stream
        # projections: dc (+)= dq Wq, dE (+)= dkv Wkv, weight / bias gradients
        for g_in, w, x_t, x, wn, bn in ((dq, W("q_weight"), c_t, c, "q_weight", "q_bias"),
                                         (dkv, W("kv_weight"), e_t, E, "kv_weight", "kv_bias")):
            if x_t in self.grad_init:
                dx = self.grads[x_t]
                K.linear_dgrad(g_in, w, dx, accumulate_into=dx, stream=st)
            else:
                K.linear_dgrad(g_in, w, self.grad_buffer(x_t), stream=st)
                self.grad_init.add(x_t)
            K.linear_wgrad(g_in, x, G(wn), accumulate=self._wgrad_acc, stream=st)
            K.colsum(g_in, G(bn), stream=st)

    # attention products straight out of the fused [M, 3H] qkv buffer
    def _scores(self, qkv, S, s):
        cfg = self.cfg
        d, A, H, b = cfg.head_dim, cfg.heads, cfg.hidden, self.b
        K.gemm_raw(M=s, N=s, K=d, A=qkv, lda=3 * H, a_s=(d, s * 3 * H), B=qkv[:, H:], ldb=3 * H,
                   b_s=(d, s * 3 * H), batch1=A, batch2=b, Cout=S, ldc=s,
                   c_s=(s * s, A * s * s), stream=self.stream)

    def _pv(self, P, qkv, O, s):
        cfg = self.cfg
        d, A, H, b = cfg.head_dim, cfg.heads, cfg.hidden, self.b
        K.gemm_raw(M=s, N=d, K=s, A=P, lda=s, a_s=(s * s, A * s * s), B=qkv[:, 2 * H:], ldb=3 * H,
                   b_mn=True, b_s=(d, s * 3 * H), batch1=A, batch2=b, Cout=O, ldc=H,
                   c_s=(d, s * H), stream=self.stream)

    # ---- backward ------------------------------------------------------------------

    def grad_buffer(self, tid: str) -> torch.Tensor:
        """Gradient buffer for tensor tid (allocated on first use)."""
        if tid not in self.grads:
            shape, dt = self._spec(tid)
            self.grads[tid] = torch.empty(shape, dtype=BF16, device=self.device)
        return self.grads[tid]

    def grad_like(self, tid: str) -> torch.Tensor:
        """A fresh bf16 buffer shaped like tensor tid (receive buffer for a grad)."""
        shape, _ = self._spec(tid)
        return torch.empty(shape, dtype=BF16, device=self.device)

    def set_recv_grad(self, tid: str, t: torch.Tensor) -> None:
        self.grads[tid] = t
        self.grad_init.add(tid)

    def _contribute_identity(self, tid: str, src: torch.Tensor) -> None:
        """grad[tid] += src, aliasing src when grad[tid] is still empty."""
        if tid not in self.grad_init:
            self.grads[tid] = src
            self.grad_init.add(tid)
            if self.cnn:
                self.shared_grads.add(tid)
        else:
            dst = self._own(tid) if self.cnn else self.grads[tid]
            K.add(dst, src, dst, stream=self.stream)

    def backward(self, mb: int) -> Dict[str, torch.Tensor]:
        """Backward of micro-batch mb.  Output-boundary grads must have been handed
        in with set_recv_grad.  Returns the grads of the recv (input-boundary) tensors."""
        st = self.stream
        slot = self.slot_of(mb)
        assert self.slot_mb[slot] == mb, "slot reused before its backward"
        ver = self.params.pinned(mb)
        with torch.cuda.stream(st):
            self._drop_leftovers()
            self._recv_mb = 0
            if not self._wgrad_acc:
                self.params.zero_accum_grads(stream=st)
            # swap-ins in first-use order (backward runs right to left), kept
            # `swap_lookahead` tensors ahead of the node that needs them
            queue = sorted(self.swap_ids, key=lambda t: (-self.bwd_first.get(t, -1), t))
            issued: Set[str] = set()
            for t, (buf, done) in self.prefetched.items():  # started by the last backward
                self.live[t] = buf
                self.swap_in_done[t] = done
                issued.add(t)
                queue.remove(t)
            self.prefetched = {}

            def issue_next() -> None:
                t = queue.pop(0)
                if t not in self.live:
                    self._swap_in(t, slot)
                issued.add(t)

            def prefetch(upto: int) -> None:
                while queue and sum(1 for t in issued if t in self.live) < upto:
                    issue_next()

            prefetch(self.swap_lookahead)
            pos = {n.id: i for i, n in enumerate(self.nodes)}
            for n in reversed(self.nodes):
                for t in self.bwd_reads[n.id]:
                    if t in self.live and t not in self.swap_in_done:
                        continue
                    if t in self.swap_ids:
                        while t not in issued:
                            if not queue:
                                raise RuntimeError(f"stage {self.stage}: swap-in of {t} never issued")
                            issue_next()
                        if t in self.swap_in_done:
                            s0 = self._stat_event(st)
                            st.wait_event(self.swap_in_done.pop(t))
                            if s0 is not None:  # compute-stream time spent waiting on the H2D
                                self.memstats["stall"].append((s0, self._stat_event(st)))
                    elif t not in self.live:  # recompute: replay its producer chain now
                        r0 = self._stat_event(st)
                        self._alloc_live(t)
                        for i in self.chains[t]:
                            self._node_fwd_replay(self.all_nodes[i], slot, ver)
                        for e in [e for e in self.live if e in self.ephemeral]:
                            del self.live[e]  # chain intermediates
                        if r0 is not None:
                            self.memstats["recompute"].append((r0, self._stat_event(st)))
                if self.node_timer is not None:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                self._node_bwd(n, slot, ver)
                if self.node_timer is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(st)
                    self.node_timer.append((n.id, "bwd", e0, e1))
                for t in self.bwd_reads[n.id]:
                    if self.bwd_last.get(t) == pos[n.id] and t in self.live:
                        del self.live[t]
                # n's output gradient is consumed: drop it (memory is recycled once
                # every alias is gone, in compute-stream order)
                self.grads.pop(out_tid(n.id), None)
                prefetch(self.swap_lookahead)
            out = {t: self.grads[t] for t in self.recv_ids if t in self.grads}
            self._prefetch_next(mb)
        return out

    def _prefetch_next(self, mb: int) -> None:
        """Start the H2D of micro-batch mb+1's first swapped tensors (up to
        prefetch_budget bytes) if its forward has run (1F1B: it has, whenever
        mb+1 <= mb + w - 1)."""
        if not self.prefetch_budget or self.sync or not self.swap_ids:
            return
        nxt = mb + 1
        slot = self.slot_of(nxt)
        if self.slot_mb[slot] != nxt:
            return
        budget = self.prefetch_budget
        for t in sorted(self.swap_ids, key=lambda t: (-self.bwd_first.get(t, -1), t)):
            size = self.host[t][slot].numel() * self.host[t][slot].element_size()
            if size > budget:
                break
            self._swap_in(t, slot, early=True)
            budget -= size

    def finish_backward(self, mb: int) -> None:
        """Optimizer step after micro-batch mb's backward (PipeDream per-micro-batch
        update); writes the next weight version into the retiring slot.  Under the
        sync schedule the gradients only accumulate; `optimizer_step` applies them."""
        if self.sync:
            self.params.version_of.pop(mb, None)
            self.params.users[0].discard(mb)
            self._wgrad_acc = True
        else:
            dst = self.params.retire(mb)
            with torch.cuda.stream(self.stream):
                self.params.adamw(dst, self.opt, stream=self.stream)
        self.grads = {}
        self.grad_init = set()
        self._skip_bwd = set()
        self._bias_done = set()
        self.shared_grads = set()

    def dp_grads(self) -> List[torch.Tensor]:
        """Tensors a data-parallel all-reduce sums before the optimizer step: the
        stage's flat fp32 weight gradient (runtime/distributed.py)."""
        return [self.params.grad]

    def optimizer_step(self) -> None:
        """Sync schedule: one AdamW step over the gradients accumulated by the
        iteration's m backwards (already averaged by the loss-gradient scale)."""
        if not self.sync:
            return
        if self.params.version_of:
            raise RuntimeError("optimizer step with micro-batches still in flight")
        with torch.cuda.stream(self.stream):
            self.params.adamw(0, self.opt, stream=self.stream)
        self._wgrad_acc = False

    def _node_fwd_replay(self, n: NodeDef, slot: int, ver: int) -> None:
        # outputs of a replayed node land in a live buffer if evicted, else in
        # their normal home (slot buffer); ephemeral ones in a live buffer that
        # the backward drops once the chain is replayed
        for t in [out_tid(n.id)] + self.self_tids(n):
            if (t in self.evicted or t in self.ephemeral) and t not in self.live:
                self._alloc_live(t)
        self._node_fwd(n, slot, ver, "bwd")

    def _node_bwd(self, n: NodeDef, slot: int, ver: int) -> None:
        cfg, M, H = self.cfg, self.M, self.cfg.hidden
        st = self.stream
        P = self.params
        W = lambda pn: P.weight(ver, f"{n.id}.{pn}")
        G = lambda pn: P.gradv(f"{n.id}.{pn}")
        k = n.kind
        tid = out_tid(n.id)
        if k == "head":
            dlog = self.buf(tid, slot, "bwd")
            x = self.buf(out_tid(n.inputs[0]), slot, "bwd")
            dx_t = out_tid(n.inputs[0])
            dx = self.grad_buffer(dx_t)
            K.linear_dgrad(dlog, W("weight"), dx, accumulate_into=dx if dx_t in self.grad_init else None,
                           stream=st)
            self.grad_init.add(dx_t)
            K.linear_wgrad(dlog, x, G("weight"), accumulate=self._wgrad_acc, stream=st)
            return
        if tid not in self.grad_init:
            return  # nothing flows into this node (cannot happen for a connected graph)
        dy = self.grads[tid]
        if k == "embed":
            off, rows = self.id_offset[n.id], node_rows(cfg, n, self.b)
            K.embed_bwd(self.ids[slot][off:off + rows], dy, G("tok"), G("pos"), n.seq or cfg.seq,
                        stream=st)
        elif k == "ln":
            x_t = out_tid(n.inputs[0])
            x = self.buf(x_t, slot, "bwd")
            stats = self.buf(stats_tid(n.id), slot, "bwd")
            lin = self.ln_bias_of.get(n.id)
            dbias = P.gradv(f"{lin}.bias") if lin is not None else None
            if x_t in self.grad_init:
                dx = self.grads[x_t]
                K.layernorm_bwd_fused(dy, x, W("gamma"), stats[0], stats[1], dx, G("gamma"),
                                      G("beta"), dx_add=dx, dbias=dbias, stream=st)
            else:
                dx = self.grad_buffer(x_t)
                K.layernorm_bwd_fused(dy, x, W("gamma"), stats[0], stats[1], dx, G("gamma"),
                                      G("beta"), dbias=dbias, stream=st)
                self.grad_init.add(x_t)
            if lin is not None:
                self._bias_done.add(lin)
        elif k in ("linear", "linear_res"):
            x_t = out_tid(n.inputs[0])
            x = self.buf(x_t, slot, "bwd")
            g_id = self.bwd_gelu_of.get(n.id)
            if g_id is not None and x_t not in self.grad_init:
                # fused GELU backward: the dgrad epilogue multiplies by gelu'(f) and
                # lands in f's gradient; the gelu node's own backward is skipped
                f_t = out_tid(self.node_by_id[g_id].inputs[0])
                df = self.grad_buffer(f_t)
                fc1 = self.gelu_bias_of.get(n.id)
                dbias = P.gradv(f"{fc1}.bias") if fc1 is not None else None
                if dbias is not None and dbias.data_ptr() % 8:
                    dbias = None  # the fused column sums need an 8-byte aligned f32 target
                K.linear_dgrad(dy, W("weight"), df, gelu_of=self.buf(f_t, slot, "bwd"), dbias=dbias,
                               stream=st)
                if dbias is not None:
                    self._bias_done.add(fc1)
                self.grad_init.add(f_t)
                self._skip_bwd.add(g_id)
            elif x_t in self.grad_init:
                dx = self.grads[x_t]
                K.linear_dgrad(dy, W("weight"), dx, accumulate_into=dx, stream=st)
            else:
                dx = self.grad_buffer(x_t)
                K.linear_dgrad(dy, W("weight"), dx, stream=st)
                self.grad_init.add(x_t)
            K.linear_wgrad(dy, x, G("weight"), accumulate=self._wgrad_acc, stream=st)
            if n.id not in self._bias_done:
                K.colsum(dy, G("bias"), stream=st)
            if k == "linear_res":
                self._contribute_identity(out_tid(n.inputs[1]), dy)
        elif k == "gelu":
            if n.id in self._skip_bwd:
                return
            x_t = out_tid(n.inputs[0])
            x = self.buf(x_t, slot, "bwd")
            assert x_t not in self.grad_init
            K.gelu_bwd(dy, x, dy, stream=st)  # in place: dy buffer becomes df
            self.grads[x_t] = dy
            self.grad_init.add(x_t)
        elif k == "add":
            self._contribute_identity(out_tid(n.inputs[0]), dy)
            self._contribute_identity(out_tid(n.inputs[1]), dy)
        elif k == "attn":
            P_t, qkv_t = out_tid(n.inputs[0]), out_tid(n.inputs[1])
            Pm = self.buf(P_t, slot, "bwd")
            qkv = self.buf(qkv_t, slot, "bwd")
            dP = self.grad_buffer(P_t)
            dqkv = self.grad_buffer(qkv_t)
            s, d, A, b = n.seq or cfg.seq, cfg.head_dim, cfg.heads, self.b
            # dP = dO V^T : A = dO (K-major over d), B = V (K-major over d)
            K.gemm_raw(M=s, N=s, K=d, A=dy, lda=H, a_s=(d, s * H), B=qkv[:, 2 * H:], ldb=3 * H,
                       b_s=(d, s * 3 * H), batch1=A, batch2=b, Cout=dP, ldc=s,
                       c_s=(s * s, A * s * s), stream=st)
            # dV = P^T dO : A = P^T (MN-major), B = dO (MN-major, d contiguous)
            K.gemm_raw(M=s, N=d, K=s, A=Pm, lda=s, a_mn=True, a_s=(s * s, A * s * s), B=dy, ldb=H,
                       b_mn=True, b_s=(d, s * H), batch1=A, batch2=b, Cout=dqkv[:, 2 * H:],
                       ldc=3 * H, c_s=(d, s * 3 * H), stream=st)
            self.grad_init.add(P_t)
        elif k == "attn_fused":
            qkv_t = out_tid(n.inputs[0])
            assert qkv_t not in self.grad_init
            dqkv = self.grad_buffer(qkv_t)
            # the QKV projection's bias gradient (column sums of dqkv) is accumulated
            # by the attention backward itself when the attention is its only reader
            lin = self.attn_bias_of.get(n.id)
            dbias = P.gradv(f"{lin}.bias") if lin is not None else None
            if dbias is not None and dbias.data_ptr() % 16:
                dbias = None
            K.attn_bwd(self.buf(qkv_t, slot, "bwd"), self.buf(tid, slot, "bwd"), dy,
                       self.buf(stats_tid(n.id), slot, "bwd"), dqkv, self.b, n.seq or cfg.seq,
                       cfg.heads, n.causal, dbias=dbias, stream=st)
            if dbias is not None:
                self._bias_done.add(lin)
            self.grad_init.add(qkv_t)
        elif k == "xattn":
            self._xattn_bwd(n, dy, slot, W, G)
        elif k == "score":
            qkv_t = out_tid(n.inputs[0])
            Pm = self.buf(tid, slot, "bwd")
            qkv = self.buf(qkv_t, slot, "bwd")
            dqkv = self.grads[qkv_t]
            s, d, A, b = n.seq or cfg.seq, cfg.head_dim, cfg.heads, self.b
            K.softmax_bwd(Pm, dy, dy, 1.0 / math.sqrt(d), stream=st)  # dy := dS (pre-scale folded)
            # dQ = dS K : A = dS (K-major over keys), B = K (MN-major, d contiguous)
            K.gemm_raw(M=s, N=d, K=s, A=dy, lda=s, a_s=(s * s, A * s * s), B=qkv[:, H:], ldb=3 * H,
                       b_mn=True, b_s=(d, s * 3 * H), batch1=A, batch2=b, Cout=dqkv, ldc=3 * H,
                       c_s=(d, s * 3 * H), stream=st)
            # dK = dS^T Q : A = dS^T (MN-major), B = Q (MN-major)
            K.gemm_raw(M=s, N=d, K=s, A=dy, lda=s, a_mn=True, a_s=(s * s, A * s * s), B=qkv, ldb=3 * H,
                       b_mn=True, b_s=(d, s * 3 * H), batch1=A, batch2=b, Cout=dqkv[:, H:],
                       ldc=3 * H, c_s=(d, s * 3 * H), stream=st)
            self.grad_init.add(qkv_t)
        elif self.cnn:
            self._cnn_bwd(n, dy, slot, W, G)
        else:
            raise ValueError(k)
