"""Measure one stage's memory plan executing on the B200.

The planner charges a stage's memory optimisation to its backward
(`bwd += added_time`, reference simulate.py:136-138): a swap costs its window
overrun (memopt.py:137-143), a recompute the forward time of its producer
chain.  `probe_stage` runs stage x of a plan *alone on its GPU* -- its real
executor, weights, w = l-x+1 weight versions and activation slots, its real
1F1B op list (`async_ops`) with synthetic boundary activations / gradients
standing in for the neighbours -- under a per-GPU allocator cap, with the
swap engine and recompute replay instrumented (StageExecutor.memstats), and
returns what the model predicted beside what ran:

* forward / backward time per micro-batch (CUDA events on the compute
  stream) vs the profile's segment times, + added_time for the backward;
* swap-in stall: compute-stream time spent waiting for an H2D prefetch;
* recompute: compute-stream time of the replayed producer chains, vs the
  plan's recompute overhead;
* D2H / H2D bytes and the achieved GB/s of the copy-stream transfers;
* the stage's device peak (max_memory_allocated above what was resident
  before the stage was built) vs the planner's sched_peak and the cap.
"""

from __future__ import annotations

import gc
from typing import Optional

import torch

from .. import planner as P
from .._lib import init_device
from ..kernels import release_workspaces
from ..planner.schedule import async_ops
from .model import TransformerConfig, build_nodes, init_params
from .stage import StageExecutor


def probe_stage(model: TransformerConfig, g, plan, x: int, b: int, *, cap: Optional[int] = None,
                micro_batches: Optional[int] = None, device: int = 0, init=None,
                swap_knobs: Optional[dict] = None, use_arena: bool = False) -> dict:
    dev = torch.device("cuda", device)
    init_device(device)
    l = len(plan.stages)
    lo, hi = P.stage_bounds(plan.cuts, len(g))[x - 1]
    w = l - x + 1
    m = micro_batches or max(2 * w, w + 2)
    total = torch.cuda.get_device_properties(device).total_memory
    gc.collect()
    torch.cuda.synchronize(device)
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated(device)
    torch.cuda.reset_peak_memory_stats(device)
    arena = None
    if cap is not None and use_arena:  # the stage's own cap-sized arena (runtime/arena.py)
        from .arena import StageArena
        arena = StageArena(device, cap)
    elif cap is not None:
        torch.cuda.set_per_process_memory_fraction(min(1.0, (cap + base) / total), device)
    ex = None
    import contextlib
    scope = contextlib.ExitStack()
    if arena is not None:
        scope.enter_context(arena.active())
    try:
        stream = torch.cuda.Stream(device=dev)
        ex = StageExecutor(cfg=model, g=g, nodes=build_nodes(model), lo=lo, hi=hi, stage=x, stages=l,
                           micro_batch=b, memopt=plan.memopt[x - 1],
                           init=init if init is not None else init_params(model, 0),
                           device=dev, stream=stream)
        ex.memstats = {"d2h": [], "h2d": [], "stall": [], "recompute": []}
        for k, v in (swap_knobs or {}).items():  # d2h_budget, prefetch_budget, swap_lookahead
            setattr(ex, k, v)
        gen = torch.Generator(device=dev).manual_seed(x)
        # harness inputs: two micro-batches, cycled, and only on the stages that
        # read them (the stage itself keeps its w input slots, like in a run)
        ishape, idt = model.input_spec(b)
        n_in = min(m, 2)
        ids = labels = None
        if ex.needs_ids:
            if idt == torch.int32:
                ids = torch.randint(0, model.vocab, (n_in,) + tuple(ishape), device=dev, dtype=idt,
                                    generator=gen)
            else:  # CNN images
                ids = torch.randn((n_in,) + tuple(ishape), device=dev, generator=gen).to(idt)
        if ex.is_last:
            labels = torch.randint(0, model.vocab, (n_in, b * model.out_tokens), device=dev,
                                   dtype=torch.int32, generator=gen)
        loss = torch.zeros(m, device=dev)
        ops = []
        with torch.cuda.stream(stream):
            for kind, j, _ in async_ops(l, m, x):
                if kind == "fwd":
                    for tid in ex.recv_ids:
                        buf = ex.recv_buffer(tid, j)
                        if buf.is_floating_point():
                            buf.normal_(0, 1, generator=gen)
                else:
                    for tid in ex.send_ids:
                        gbuf = ex.grad_like(tid)
                        gbuf.normal_(0, 1e-3, generator=gen)
                        ex.set_recv_grad(tid, gbuf)
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if kind == "fwd":
                    ex.forward(j, ids=ids[(j - 1) % n_in] if ex.needs_ids else None,
                               labels=labels[(j - 1) % n_in] if ex.is_last else None,
                               loss_out=loss[j - 1:j] if ex.is_last else None)
                else:
                    ex.backward(j)
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                ops.append((kind, j, e0, e1))
                if kind == "bwd":  # the PipeDream update, outside the modelled t_b
                    ex.finish_backward(j)
                    e2 = torch.cuda.Event(enable_timing=True)
                    e2.record(stream)
                    ops.append(("opt", j, e1, e2))
        torch.cuda.synchronize(device)
        peak = torch.cuda.max_memory_allocated(device) - base
        if arena is not None:  # the arena's high-water mark (allocator segments)
            peak = arena.stats()[1]
        st = ex.memstats

        def span_us(pairs):
            return sum(a.elapsed_time(b) for a, b in pairs) * 1e3

        def rate(rows):
            nbytes = sum(r[0] for r in rows)
            us = sum(r[1].elapsed_time(r[2]) for r in rows) * 1e3
            return {"bytes_per_mb": nbytes // m, "copy_us_per_mb": round(us / m, 1),
                    "GBps": round(nbytes / us / 1e3, 2) if us > 0 else None}

        # the first backward pays one-off costs (first touch of the gradient
        # buffers, workspace growth): steady-state means skip it
        fwd = [a.elapsed_time(b) * 1e3 for k, j, a, b in ops if k == "fwd"]
        bwd = [a.elapsed_time(b) * 1e3 for k, j, a, b in ops if k == "bwd"][1:]
        mo = plan.memopt[x - 1]
        swap_model = sum(a.overhead_us for a in mo.actions if a.kind == "swap")
        rec_model = sum(a.overhead_us for a in mo.actions if a.kind == "recompute")
        out = {
            "stage": x, "stages": l, "nodes": [lo, hi], "micro_batch": b, "micro_batches": m,
            "swap_knobs": {"d2h_budget": ex.d2h_budget, "prefetch_budget": ex.prefetch_budget,
                           "swap_lookahead": ex.swap_lookahead},
            "actions": {"swap": sum(a.kind == "swap" for a in mo.actions),
                        "recompute": sum(a.kind == "recompute" for a in mo.actions),
                        "bytes_saved": mo.bytes_saved},
            "fwd_us": {"model": g.segment_fwd_time(lo, hi), "measured": round(sum(fwd) / len(fwd), 1)},
            "bwd_us": {"model_without_memopt": g.segment_bwd_time(lo, hi),
                       "model": g.segment_bwd_time(lo, hi) + mo.added_time,
                       "measured": round(sum(bwd) / max(1, len(bwd)), 1)},
            "optimizer_us": round(sum(a.elapsed_time(b) * 1e3 for k, j, a, b in ops if k == "opt") / m, 1),
            "added_time_us": {"model": mo.added_time, "model_swap": swap_model,
                              "model_recompute": rec_model,
                              "measured_stall_per_mb": round(span_us(st["stall"]) / m, 1),
                              "measured_recompute_per_mb": round(span_us(st["recompute"]) / m, 1)},
            "d2h": rate(st["d2h"]), "h2d": rate(st["h2d"]),
            "peak_bytes": {"measured": peak, "planner_sched_peak": plan.stages[x - 1].sched_peak,
                           "cap": cap},
        }
        return out
    finally:
        del ex
        release_workspaces()
        gc.collect()
        scope.close()
        if arena is not None:
            arena.close()
        gc.collect()
        torch.cuda.synchronize(device)
        torch.cuda.empty_cache()
        torch.cuda.set_per_process_memory_fraction(1.0, device)


def heaviest_stage(plan) -> int:
    """1-based stage evicting the most bytes."""
    return max(range(1, len(plan.stages) + 1), key=lambda x: (plan.memopt[x - 1].bytes_saved, -x))
