"""Max trainable micro-batch under a per-GPU memory cap (the second half of
BASELINE.json's metric; SURVEY.md 8(d) "Max-batch metric").

For each micro-batch size b:
  1. build the model's profile graph at b (runtime/graph.py; analytic or
     measured node times),
  2. plan it with the planner at the cap minus the memory the planner's model
     does not see (fp32 master / Adam m / Adam v / grad: 16 B per parameter,
     plus a fixed workspace reserve),
  3. run every stage of the plan *on the GPU under the cap*: the stage's own
     executor (weights, w = l-x+1 weight versions and activation slots, the
     plan's swap / recompute actions) runs its real 1F1B op list for
     m = w + 1 micro-batches with synthetic boundary activations / gradients
     standing in for its neighbours.  The cap is enforced on the caching
     allocator (torch.cuda.set_per_process_memory_fraction); an allocation
     beyond it raises OutOfMemoryError.
b is trainable iff the planner returns a plan and every stage completes; for
the planned strategies a stage that runs out of memory on the GPU sends b back
to the planner with a 10% / 20% smaller capacity first (`max_batch`, measured-
memory feedback for what the profile's memory model leaves out).

The baseline is the even-compute split: `compute_balanced` cuts with empty
memopt plans (`plan_from_cuts(..., require_feasible=False)`, as the reference
CLI's `compare` builds it, cli.py:276-300), checked the same way.
"""

from __future__ import annotations

import gc
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import torch

from .. import planner as P
from .._lib import init_device
from ..kernels import release_workspaces
from ..planner.memplan import MemOptPlan
from ..planner.schedule import async_ops
from .graph import profile_graph
from .model import TransformerConfig, build_nodes, init_params
from .stage import StageExecutor

GIB = 1 << 30


@dataclass
class StageCheck:
    stage: int
    ok: bool
    peak_bytes: int
    error: str = ""


@dataclass(frozen=True)
class Overhead:
    """Device bytes of a stage the planner's memory model (w x (micro_peak -
    saved), memopt.py:156-158) does not see, as a linear function of the
    stage: per_param x (bytes of one bf16 weight version, the profile's m_p)
    + per_act x (the stage's largest activation) + const.  What it stands for:
    fp32 master / Adam m / Adam v / grad (8 bytes per m_p byte), backward
    gradient buffers, the D2H back-pressure window, workspaces and allocator
    slack."""

    per_param: float = 8.0
    per_act: float = 2.0
    const: int = 3 * GIB // 2
    source: str = "hand-calibrated (round 1: 16 B/param + 2 x largest activation + 1.5 GiB)"

    def to_doc(self) -> dict:
        return {"per_param": self.per_param, "per_act": self.per_act, "const": self.const,
                "source": self.source}


DEFAULT_OVERHEAD = Overhead()


def _stage_features(g, lo: int, hi: int) -> Tuple[int, int]:
    return g.segment_params(lo, hi), max(g.nodes[k].m_a for k in range(lo, hi + 1))


def stage_overhead(model: TransformerConfig, g, lo: int, hi: int, b: int,
                   overhead: Overhead = DEFAULT_OVERHEAD) -> int:
    params, largest = _stage_features(g, lo, hi)
    return int(overhead.per_param * params + overhead.per_act * largest + overhead.const)


def optimizer_reserve(model: TransformerConfig, g, stages: int, cuts=None, b: int = 1,
                      overhead: Overhead = DEFAULT_OVERHEAD) -> int:
    """Max stage_overhead over the stages of `cuts` (default: compute-balanced)."""
    if cuts is None:
        cuts = P.compute_balanced(g, 0, len(g) - 1, [1] * stages).positions
    bounds = P.stage_bounds(P.Cut(tuple(cuts)), len(g))
    return max(stage_overhead(model, g, lo, hi, b, overhead) for lo, hi in bounds)


def calibrate_overhead(model: TransformerConfig, stages: int, device: int = 0,
                       sizes: Tuple[int, ...] = (1, 2), times=None) -> Tuple[Overhead, List[dict]]:
    """Fit `Overhead` to measured stage peaks: every stage of the
    compute-balanced split (no memopt) runs alone on the GPU at each micro-batch
    size in `sizes` (runtime/memprobe.py); the unmodelled bytes (measured peak
    - the planner's sched_peak) are least-squares fitted on (m_p bytes,
    largest activation, 1), and the constant is raised by the largest
    under-prediction so the fit bounds every measurement from above."""
    import numpy as np
    from .memprobe import probe_stage
    rows, ys, pts = [], [], []
    init = init_params(model, 0)
    for b in sizes:
        g = profile_graph(model, b, times=times)
        ample = P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=1 << 62,
                             bandwidth=1 << 40)
        plan = P.plan_from_cuts(g, ample, P.compute_balanced(g, 0, len(g) - 1, [1] * stages).positions)
        for x, (lo, hi) in enumerate(P.stage_bounds(plan.cuts, len(g)), start=1):
            r = probe_stage(model, g, plan, x, b, device=device, micro_batches=stages - x + 2, init=init)
            extra = r["peak_bytes"]["measured"] - plan.stages[x - 1].sched_peak
            params, largest = _stage_features(g, lo, hi)
            rows.append([params, largest, 1.0])
            ys.append(extra)
            pts.append({"b": b, "stage": x, "measured_peak": r["peak_bytes"]["measured"],
                        "sched_peak": plan.stages[x - 1].sched_peak, "unmodelled": extra})
    A, y = np.array(rows, dtype=np.float64), np.array(ys, dtype=np.float64)
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    per_param, per_act = max(0.0, float(coef[0])), max(0.0, float(coef[1]))
    const = y - (per_param * A[:, 0] + per_act * A[:, 1])
    oh = Overhead(per_param=round(per_param, 3), per_act=round(per_act, 3), const=int(const.max()),
                  source=f"measured: {len(ys)} stage peaks at b in {list(sizes)}, least squares, "
                         f"constant raised to bound every point")
    return oh, pts


def check_stage(model: TransformerConfig, g, plan, x: int, b: int, cap: int, device: int = 0,
                micro_batches: Optional[int] = None, init=None) -> StageCheck:
    """Run stage x of `plan` alone under a `cap`-byte allocator limit."""
    dev = torch.device("cuda", device)
    init_device(device)
    l = len(plan.stages)
    lo, hi = P.stage_bounds(plan.cuts, len(g))[x - 1]
    total = torch.cuda.get_device_properties(device).total_memory
    gc.collect()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(device)
    torch.cuda.set_per_process_memory_fraction(min(1.0, cap / total), device)
    ex = None
    try:
        stream = torch.cuda.Stream(device=dev)
        ex = StageExecutor(cfg=model, g=g, nodes=build_nodes(model), lo=lo, hi=hi, stage=x,
                           stages=l, micro_batch=b, memopt=plan.memopt[x - 1],
                           init=init if init is not None else init_params(model, 0),
                           device=dev, stream=stream)
        w = l - x + 1
        m = micro_batches or (w + 1)
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
        with torch.cuda.stream(stream):
            for kind, j, _ in async_ops(l, m, x):
                if kind == "fwd":
                    for tid in ex.recv_ids:
                        buf = ex.recv_buffer(tid, j)
                        buf.normal_(0, 1, generator=gen) if buf.is_floating_point() else None
                    ex.forward(j, ids=ids[(j - 1) % n_in] if ex.needs_ids else None,
                               labels=labels[(j - 1) % n_in] if ex.is_last else None,
                               loss_out=loss[j - 1:j] if ex.is_last else None)
                else:
                    for tid in ex.send_ids:
                        gbuf = ex.grad_like(tid)
                        gbuf.normal_(0, 1e-3, generator=gen)
                        ex.set_recv_grad(tid, gbuf)
                    ex.backward(j)
                    ex.finish_backward(j)
        torch.cuda.synchronize(device)
        return StageCheck(x, True, torch.cuda.max_memory_allocated(device))
    except torch.OutOfMemoryError as e:
        return StageCheck(x, False, torch.cuda.max_memory_allocated(device), str(e).split("\n")[0][:200])
    except RuntimeError as e:  # pinned host slots for swaps beyond what the OS lets us lock
        if "pin" not in str(e).lower() and "OS call failed" not in str(e):
            raise
        return StageCheck(x, False, torch.cuda.max_memory_allocated(device),
                          "pinned host allocation failed: " + str(e).split("\n")[0][:160])
    finally:
        del ex
        release_workspaces()  # per-stream scratch of this trial's stream
        gc.collect()
        torch.cuda.synchronize(device)
        torch.cuda.empty_cache()
        torch.cuda.set_per_process_memory_fraction(1.0, device)


def host_bytes(plan, stages: int) -> List[int]:
    """Pinned host bytes per stage: w = l-x+1 slots (x 1-based, as
    StageExecutor allocates them) of every swapped tensor."""
    return [(stages - x + 1) * sum(a.size for a in m.actions if a.kind == "swap")
            for x, m in enumerate(plan.memopt, start=1)]


def plan_for_cap(model: TransformerConfig, g, stages: int, cap: int, bandwidth: int,
                 margin: float = 0.0, b: int = 1, overhead: Overhead = DEFAULT_OVERHEAD,
                 link_aware: bool = False):
    """DawnPiper plan for a per-GPU byte cap: the planner gets the cap minus
    what its memory model does not see (`stage_overhead`), re-planned with the
    reserve of the plan's own stages until every stage's overhead is covered.
    Raises InfeasibleModelError."""
    reserve = optimizer_reserve(model, g, stages, b=b, overhead=overhead)
    cfg = P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC,
                       capacity=max(1, int((cap - reserve) * (1.0 - margin))), bandwidth=bandwidth,
                       link_aware=link_aware)
    for _ in range(4):
        plan = P.plan(g, cfg)
        need = optimizer_reserve(model, g, stages, plan.cuts.positions, b=b, overhead=overhead)
        pcap = int((cap - need) * (1.0 - margin))
        if pcap >= cfg.capacity:
            break
        if pcap <= 0:
            raise P.InfeasibleModelError("stage overhead alone exceeds the cap")
        cfg = P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=pcap,
                           bandwidth=bandwidth, link_aware=link_aware)
    return plan, cfg


def try_batch(model: TransformerConfig, b: int, stages: int, cap: int, bandwidth: int,
              strategy: str, device: int = 0, times=None, run_gpu: bool = True,
              host_cap: int = 96 * GIB, margin: float = 0.0,
              overhead: Overhead = DEFAULT_OVERHEAD, timing: bool = False) -> dict:
    """One trial; `margin` shrinks the capacity handed to the planner by that
    fraction (the measured-memory feedback of `max_batch`)."""
    g = profile_graph(model, b, times=times)
    reserve = optimizer_reserve(model, g, stages, b=b, overhead=overhead)
    pcap = int((cap - reserve) * (1.0 - margin))
    rec = {"b": b, "strategy": strategy, "planner_capacity": pcap, "reserve": reserve}
    if margin:
        rec["margin"] = margin
    cfg = P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=max(1, pcap),
                       bandwidth=bandwidth)
    if pcap <= 0:
        rec.update(feasible=False, reason="optimizer state alone exceeds the cap")
        return rec
    if strategy in ("dawnpiper", "dawnpiper_link"):
        try:
            plan, cfg = plan_for_cap(model, g, stages, cap, bandwidth, margin, b, overhead,
                                     link_aware=strategy == "dawnpiper_link")
        except P.InfeasibleModelError as e:
            rec.update(feasible=False, reason=f"planner: {e}")
            return rec
        rec["planner_capacity"] = cfg.capacity
    elif strategy == "even_compute_memopt":
        # even-compute cuts + the same per-stage memopt policy (cli.py:276-300 "compute_balanced")
        cb = P.compute_balanced(g, 0, len(g) - 1, [1] * stages)
        try:
            plan = P.plan_from_cuts(g, cfg, cb.positions, require_feasible=True)
        except P.InfeasibleModelError as e:
            rec.update(feasible=False, reason=f"planner: {e}", cuts=list(cb.positions))
            return rec
    elif strategy == "even_compute":
        # even-compute cuts, no memory optimisation (PipeDream-style baseline)
        cb = P.compute_balanced(g, 0, len(g) - 1, [1] * stages)
        ample = P.PlanConfig(stages=stages, schedule=P.SCHEDULE_ASYNC, capacity=1 << 62,
                             bandwidth=bandwidth)
        plan = P.plan_from_cuts(g, ample, cb.positions)
        over = [s.stage for s in plan.stages if s.sched_peak > pcap]
        if over:
            rec.update(feasible=False, reason=f"stages {over} exceed the capacity without memopt",
                       cuts=list(plan.cuts.positions))
            return rec
    else:
        raise ValueError(strategy)
    rec["cuts"] = list(plan.cuts.positions)
    rec["actions"] = [[a.kind for a in m.actions].count("swap") for m in plan.memopt]
    rec["recomputes"] = [[a.kind for a in m.actions].count("recompute") for m in plan.memopt]
    rec["sched_peak_gib"] = [round(s.sched_peak / GIB, 2) for s in plan.stages]
    hb = host_bytes(plan, stages)
    rec["host_pinned_gib"] = [round(h / GIB, 1) for h in hb]
    if max(hb) > host_cap:
        # swap slots live in pinned host memory, which the planner does not model
        rec.update(feasible=False, reason=f"pinned host memory {max(hb) / GIB:.1f} GiB > {host_cap / GIB:.0f} GiB per GPU")
        return rec
    if not run_gpu:
        rec["feasible"] = True
        return rec
    init = init_params(model, 0)
    if timing:
        return _timed_stages(rec, model, g, plan, b, cap, device, init)
    checks = [check_stage(model, g, plan, x, b, cap, device, init=init) for x in range(1, stages + 1)]
    rec["stage_peak_gib"] = [round(c.peak_bytes / GIB, 2) for c in checks]
    bad = [c for c in checks if not c.ok]
    rec["feasible"] = not bad
    if bad:
        rec["reason"] = f"stage {bad[0].stage} OOM on GPU: {bad[0].error}"
    return rec


def _timed_stages(rec: dict, model, g, plan, b: int, cap: int, device: int, init) -> dict:
    """Every stage alone on the GPU under the cap with timing (memprobe), and
    the 1F1B steady-state throughput those stage times give on l GPUs: one
    micro-batch per bottleneck-stage period (forward + backward + the
    per-micro-batch AdamW of the slowest stage; boundary transfers over
    NVLink are overlapped and not charged)."""
    from .memprobe import probe_stage
    per = []
    for x in range(1, len(plan.stages) + 1):
        try:
            # the same op list length as the feasibility check (w + 1 micro-batches)
            r = probe_stage(model, g, plan, x, b, cap=cap, device=device, init=init,
                            micro_batches=len(plan.stages) - x + 2)
        except torch.OutOfMemoryError as e:
            rec.update(feasible=False, reason=f"stage {x} OOM on GPU: {str(e).splitlines()[0][:160]}")
            return rec
        per.append({"stage": x, "fwd_us": r["fwd_us"]["measured"], "bwd_us": r["bwd_us"]["measured"],
                    "opt_us": r["optimizer_us"], "model_us": r["fwd_us"]["model"] + r["bwd_us"]["model"],
                    "stall_us": r["added_time_us"]["measured_stall_per_mb"],
                    "recompute_us": r["added_time_us"]["measured_recompute_per_mb"],
                    "peak_gib": round(r["peak_bytes"]["measured"] / GIB, 2)})
    period = max(p["fwd_us"] + p["bwd_us"] + p["opt_us"] for p in per)
    model_period = max(p["model_us"] for p in per)
    rec.update(feasible=True, stage_times=per, bottleneck_us=round(period, 1),
               samples_per_s_l_gpus=round(b * 1e6 / period, 1),
               samples_per_s_l_gpus_model=round(b * 1e6 / model_period, 1),
               stage_peak_gib=[p["peak_gib"] for p in per])
    return rec


def max_batch(model: TransformerConfig, stages: int, cap: int, bandwidth: int, strategy: str,
              b_max: int = 64, device: int = 0, log=None, host_cap: int = 96 * GIB,
              run_gpu: bool = True, margins: Tuple[float, ...] = (0.1, 0.2),
              overhead: Overhead = DEFAULT_OVERHEAD, b_start: int = 1) -> Tuple[int, List[dict]]:
    """Largest feasible b (0 if none) by doubling then bisection.

    Measured-memory feedback for the planned strategies: the planner's memory
    model (the reference's) has no term for backward gradient buffers or kernel
    scratch, so when a plan's stage runs out of memory on the GPU the same b is
    re-planned with the capacity shrunk by each of `margins` in turn before it
    counts as infeasible (the fixed even-compute split has nothing to re-plan)."""
    hist: List[dict] = []

    def ok(b: int) -> bool:
        for margin in (0.0,) + (tuple(margins) if strategy != "even_compute" else ()):
            r = try_batch(model, b, stages, cap, bandwidth, strategy, device, host_cap=host_cap,
                          run_gpu=run_gpu, margin=margin, overhead=overhead)
            hist.append(r)
            if log:
                log(r)
            if r.get("feasible"):
                return True
            if "OOM on GPU" not in r.get("reason", ""):
                return False  # planner / host-memory infeasibility: a margin cannot help
        return False

    if b_start > 1 and ok(b_start):  # resume from a size known to fit
        lo, hi, b = b_start, None, 2 * b_start
    else:
        if not ok(1):
            return 0, hist
        lo, hi, b = 1, None, 2
    while b <= b_max:
        if ok(b):
            lo = b
            b *= 2
        else:
            hi = b
            break
    if hi is None:
        return lo, hist
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if ok(mid):
            lo = mid
        else:
            hi = mid
    return lo, hist
